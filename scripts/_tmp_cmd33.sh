mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu12.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu12.log
timeout 300 python scripts/ab_env.py --strategy two_tile_sk_dp --set SKB200_PRELOAD=0 --set SKB200_PRELOAD=1 --rounds 4 --steps 20 --cool 1 --no-check > gpurun_out/ab_pre_2t.json 2>&1
for S in 1280x3840x4096 1280x3840x8192 2304x2304x8192 1024x4864x4096 2560x3840x4096; do
IFS=x read M N K <<< "$S"
timeout 300 python scripts/ab_env.py --m $M --n $N --k $K --strategy two_tile_sk_dp --set SKB200_PRELOAD=0 --set SKB200_PRELOAD=1 --rounds 3 --steps 50 --cool 0.3 --no-check > gpurun_out/ab_pre_$S.json 2>&1
done
timeout 200 python scripts/wave_drift.py --strategy two_tile_sk_dp --out gpurun_out/drift_pre_2t.npy > gpurun_out/drift_pre_2t.json 2>&1
