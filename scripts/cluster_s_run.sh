#!/bin/bash
# GPU validation of the cluster fixup's S = 3 policy (outputs under gpurun_out/cs2/):
# cluster GPU tests, config-3 / skinny sweeps on the shipped policy, then every
# 2-SM corpus shape whose pick changes and a sample of the 1-SM ones.
set -u
O=gpurun_out/cs2
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -k "cluster" > $O/pytest_cluster.log 2>&1; echo rc=$? >> $O/pytest_cluster.log
for v in 1sm 2sm; do
  timeout 600 python -m paper_2301_03598_b200.sweep --shapes skinny --variant $v --dtype bf16 \
    --strategies data_parallel,stream_k:auto --out $O/skinny_$v.csv > $O/skinny_$v.log 2>&1
  timeout 600 python -m paper_2301_03598_b200.sweep --shapes config3 --variant $v --dtype bf16 \
    --strategies data_parallel,stream_k:auto --out $O/config3_$v.csv > $O/config3_$v.log 2>&1
  timeout 600 python -m paper_2301_03598_b200.sweep --shapes config3 --variant $v --dtype fp16 \
    --strategies data_parallel,stream_k:auto --out $O/config3_${v}_fp16.csv > $O/config3_${v}_fp16.log 2>&1
done
timeout 3600 python scripts/cluster_s_validate.py --variant 2sm --max ${MAX2:-0} --out $O/validate_2sm.jsonl > $O/validate_2sm.log 2>&1
timeout 1800 python scripts/cluster_s_validate.py --variant 1sm --max ${MAX1:-600} --out $O/validate_1sm.jsonl > $O/validate_1sm.log 2>&1
