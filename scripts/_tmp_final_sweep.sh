mkdir -p gpurun_out
timeout 3300 python -m paper_2301_03598_b200.sweep --shapes corpus --dtype fp16 --strategies data_parallel,stream_k:auto --out gpurun_out/sweep_corpus_full_fp16_r01f.csv --log-every 8000 > gpurun_out/sweep_corpus_full_r01f.log 2>&1
echo rc=$?
timeout 900 python -m paper_2301_03598_b200.sweep --shapes config3 --strategies data_parallel,stream_k:auto,stream_k,two_tile_sk_dp,dp_one_tile_sk --out gpurun_out/sweep_c3_r01f.csv > gpurun_out/sweep_c3_r01f.log 2>&1
timeout 600 python -m paper_2301_03598_b200.sweep --shapes skinny --strategies data_parallel,stream_k:auto,stream_k,two_tile_sk_dp --out gpurun_out/sweep_skinny_r01f.csv > gpurun_out/sweep_skinny_r01f.log 2>&1
