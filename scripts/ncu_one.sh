#!/bin/bash
# One full ncu capture of the 4th sk_gemm launch of a bench invocation.
#   NAME=<out name> bash scripts/ncu_one.sh <bench args...>
set -u
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sk_gemm -s 3 -c 1 \
  -o gpurun_out/${NAME} python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-sweep "$@" \
  > gpurun_out/${NAME}.log 2>&1
