#!/usr/bin/env bash
# Dev tool: sweep L2 policy / raster knobs of the CTA-pair grouped GEMM.
for cfg in "4096 14336 8 4096" "2048 1408 64 4096"; do
  for pol in 0 5 15 10; do
    for r in 0 1 2 8 16; do
      echo "== cfg=$cfg POL=$pol RASTER=$r"
      POL=$pol RASTER=$r timeout 120 python tools/gemm_perf.py $cfg | tr '\n' ' ' | sed 's/  */ /g'
      echo
    done
  done
done
