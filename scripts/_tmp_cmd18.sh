mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu7.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu7.log
for TG in 1 0; do
SKB200_TILE_GROUP=$TG timeout 900 python -m paper_2301_03598_b200.sweep --shapes config3 --strategies data_parallel,stream_k:auto,stream_k,two_tile_sk_dp --out gpurun_out/sweep_c3_tg$TG.csv > gpurun_out/sweep_c3_tg$TG.log 2>&1
SKB200_TILE_GROUP=$TG timeout 1200 python -m paper_2301_03598_b200.sweep --shapes corpus --count 1000 --strategies data_parallel,stream_k:auto,stream_k --out gpurun_out/sweep_corpus1000_tg$TG.csv > gpurun_out/sweep_corpus1000_tg$TG.log 2>&1
done
