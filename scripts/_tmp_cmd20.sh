mkdir -p gpurun_out
TAG=r01c bash scripts/gpu_profile.sh
timeout 300 python scripts/fp64_compare.py > gpurun_out/fp64_cmp.json 2>&1
timeout 300 python scripts/cublas_compare.py --rounds 3 > gpurun_out/cublas_cmp2.json 2>&1
