#!/bin/bash
# Round-2 closing measurements on one B200 (outputs under gpurun_out/final/):
# GPU test suite, the default bench line, the ncu launch list + full captures of
# the 8192^3 launches, and ncu DRAM bytes of the skinny shapes' policy picks.
set -u
O=gpurun_out/final
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1; echo rc=$? >> $O/pytest.log
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
TAG=final bash scripts/gpu_profile.sh
mv gpurun_out/launches_final.* gpurun_out/prof_final_* $O/ 2>/dev/null
for v in 1sm 2sm; do
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -k regex:sk_gemm --csv --log-file $O/skinny_ncu_$v.csv \
    python scripts/skinny_launch.py --variant $v > $O/skinny_launch_$v.json 2>> $O/err.log
done
