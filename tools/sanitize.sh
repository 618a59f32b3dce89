#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the smoke step
# (2 virtual ranks, tiny shapes) and the configs[0] 8-virtual-rank step.
# Usage (GPU box): bash tools/sanitize.sh [outdir]
out=${1:-gpurun_out/sanitize}
mkdir -p "$out"
CS=/usr/local/cuda/bin/compute-sanitizer
run() {  # name tool cmd...
  local name=$1 tool=$2; shift 2
  timeout 1200 $CS --tool "$tool" --print-limit 50 --error-exitcode 9 "$@" > "$out/$name.$tool.log" 2>&1
  echo "$name $tool exit=$?" | tee -a "$out/summary.txt"
  tail -3 "$out/$name.$tool.log" >> "$out/summary.txt"
}
for tool in memcheck racecheck synccheck; do
  run smoke $tool python -c "import __graft_entry__ as g; g.smoke()"
  run tiny8 $tool python tools/sanitize_step.py ${SAN_MODE:-}
done
