o=gpurun_out/r02b; mkdir -p $o
python bench.py --config tiny --steps 20 --warmup 5 > $o/tiny.json 2> $o/tiny.err; echo tiny=$?
python bench.py --steps 20 --warmup 5 > $o/mix.json 2> $o/mix.err; echo mix=$?
python bench.py --impl reference --steps 3 --warmup 1 > $o/mix_ref.json 2> $o/mix_ref.err; echo mref=$?
python bench.py --impl reference --config tiny --steps 5 --warmup 2 > $o/tiny_ref.json 2> $o/tiny_ref.err; echo tref=$?
nproc
