#!/bin/bash
# Run on the GPU box (via gpurun): launch list + one full ncu capture per
# strategy of the default bench workload.  Outputs land in gpurun_out/.
set -u
TAG=${TAG:-r01}
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
  --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-sweep \
  > gpurun_out/launches_${TAG}.log 2>&1
for S in ${STRATS:-two_tile_sk_dp data_parallel}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sk_gemm -s 3 -c 1 \
    -o gpurun_out/prof_${TAG}_${S} python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-sweep \
    --strategy $S > gpurun_out/prof_${TAG}_${S}.log 2>&1
done
