mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_final.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo smoke rc=$?
timeout 400 python bench.py > gpurun_out/bench_final.json 2>&1; echo bench rc=$?
timeout 400 python bench.py --dtype fp64 --no-e2e --no-cpu --no-sweep > gpurun_out/bench_final_fp64.json 2>&1
TAG=r01e bash scripts/gpu_profile.sh
