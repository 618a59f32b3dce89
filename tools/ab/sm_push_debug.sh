export FSEP_COMM=sm FSEP_SPIN_TIMEOUT_MS=20000
TAG=mix_default timeout 300 python tools/ab/sm_push_debug.py
TAG=mix_nosplit FSEP_RESTORE_SPLIT=0 timeout 300 python tools/ab/sm_push_debug.py
TAG=mix_148cta FSEP_PUSH_CTAS=148 timeout 300 python tools/ab/sm_push_debug.py
TAG=mix_8cta FSEP_PUSH_CTAS=8 timeout 300 python tools/ab/sm_push_debug.py
TAG=small HH=1024 FF=2048 timeout 300 python tools/ab/sm_push_debug.py
FSEP_COMM=ce TAG=ce_mix timeout 300 python tools/ab/sm_push_debug.py
