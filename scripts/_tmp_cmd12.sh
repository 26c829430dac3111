mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu3.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu3.log
for S in 1024x1024x32768 512x512x65536 1024x1024x8192 1280x3840x4096 2304x2304x8192 8192x8192x8192; do
IFS=x read M N K <<< "$S"
timeout 300 python scripts/ab_env.py --m $M --n $N --k $K --strategy two_tile_sk_dp --set SKB200_COOP=0 --set SKB200_COOP=1 --rounds 3 --steps 50 --cool 0.5 > gpurun_out/ab_coop_$S.json 2>&1
timeout 300 python scripts/ab_env.py --m $M --n $N --k $K --strategy stream_k --set SKB200_COOP=0 --set SKB200_COOP=1 --rounds 3 --steps 50 --cool 0.5 > gpurun_out/ab_coopsk_$S.json 2>&1
done
