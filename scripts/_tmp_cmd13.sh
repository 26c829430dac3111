mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu4.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu4.log
for S in 1024x1024x32768 512x512x65536 1024x1024x8192 1280x3840x4096 768x768x16384 256x512x65536; do
IFS=x read M N K <<< "$S"
timeout 300 python scripts/ab_env.py --m $M --n $N --k $K --strategy stream_k --set SKB200_COOP=0 --set SKB200_COOP=2 --set SKB200_COOP=4 --set SKB200_COOP=6 --set SKB200_COOP=8 --set SKB200_COOP=12 --rounds 3 --steps 50 --cool 0.3 > gpurun_out/ab_coopmin_$S.json 2>&1
done
