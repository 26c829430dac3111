mkdir -p gpurun_out
timeout 900 python -m paper_2301_03598_b200.sweep --shapes config3 --strategies data_parallel,stream_k:auto --out gpurun_out/sweep_c3_coopm2.csv > gpurun_out/sweep_c3_coopm2.log 2>&1
timeout 1200 python -m paper_2301_03598_b200.sweep --shapes corpus --count 1000 --strategies data_parallel,stream_k:auto --out gpurun_out/sweep_corpus1000_coopm2.csv > gpurun_out/sweep_corpus1000_coopm2.log 2>&1
