#!/bin/bash
# BASELINE config 5 on the shipped policy: the full 32,824-shape FP16 corpus (seed 0), 2-SM
# kernel, DP vs stream_k:auto, every row verified; four chunks (outputs under gpurun_out/$1/).
set -u
O=gpurun_out/${1:-corpus}
mkdir -p $O
for c in 0 1 2 3; do
  timeout 2400 python -m paper_2301_03598_b200.sweep --shapes corpus --offset $((c * 8206)) --count 8206 \
    --variant 2sm --dtype fp16 --strategies data_parallel,stream_k:auto \
    --out $O/corpus_chunk$c.csv > $O/chunk$c.json 2> $O/chunk$c.err
done
