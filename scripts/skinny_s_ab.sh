mkdir -p gpurun_out/r04b
timeout 1200 python scripts/skinny_ab.py --shapes all --coop -1 --variants 1sm,2sm \
  --strategies data_parallel,stream_k:auto,stream_k,fixed_split:2,fixed_split:3,fixed_split:4,fixed_split:5,fixed_split:6,fixed_split:7,fixed_split:8,fixed_split:9,fixed_split:12 \
  > gpurun_out/r04b/skinny_s_ab.jsonl 2> gpurun_out/r04b/err.log
python -c "import paper_2301_03598_b200 as sk; print({v:{S: sk.cluster_capacity(S, getattr(sk.Variant, v)) for S in range(2,9)} for v in ('OneSM','TwoSM')})" > gpurun_out/r04b/caps.txt 2>&1
