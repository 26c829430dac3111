mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu8.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu8.log
timeout 300 python bench.py > gpurun_out/bench_tg.json 2>&1
tail -c 1800 gpurun_out/bench_tg.json
