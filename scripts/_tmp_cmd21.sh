mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cooperative or smoke or auto" > gpurun_out/pytest_gpu9.log 2>&1; echo pytest rc=$?
timeout 900 python -m paper_2301_03598_b200.sweep --shapes config3 --strategies data_parallel,stream_k:auto,stream_k,two_tile_sk_dp --out gpurun_out/sweep_c3_final.csv > gpurun_out/sweep_c3_final.log 2>&1
timeout 1200 python -m paper_2301_03598_b200.sweep --shapes corpus --count 1000 --strategies data_parallel,stream_k:auto --out gpurun_out/sweep_corpus1000_final.csv > gpurun_out/sweep_corpus1000_final.log 2>&1
