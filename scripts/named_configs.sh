#!/bin/bash
# Named BASELINE configs on the shipped policy, every row verified (outputs under gpurun_out/$1/):
# config 3 (BF16 + FP16, both kernels), config 4 (FP64), the skinny set (both kernels).
set -u
O=gpurun_out/${1:-named}
mkdir -p $O
for v in 2sm 1sm; do
  for dt in bf16 fp16; do
    timeout 900 python -m paper_2301_03598_b200.sweep --shapes config3 --variant $v --dtype $dt \
      --strategies data_parallel,stream_k:auto,stream_k,two_tile_sk_dp --out $O/config3_${v}_$dt.csv > $O/config3_${v}_$dt.json 2> $O/err.log
  done
  timeout 900 python -m paper_2301_03598_b200.sweep --shapes skinny --variant $v --dtype bf16 \
    --strategies data_parallel,stream_k:auto --out $O/skinny_$v.csv > $O/skinny_$v.json 2>> $O/err.log
done
timeout 1500 python -m paper_2301_03598_b200.sweep --shapes config4 --variant 1sm --dtype fp64 \
  --strategies data_parallel,stream_k:auto,stream_k,two_tile_sk_dp --out $O/config4_fp64.csv > $O/config4_fp64.json 2>> $O/err.log
