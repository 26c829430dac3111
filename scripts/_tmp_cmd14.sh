mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu5.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu5.log
for S in 1024x1024x32768 512x512x65536 1024x1024x8192 1280x3840x4096 768x768x16384 256x512x65536 1024x768x24576; do
IFS=x read M N K <<< "$S"
timeout 300 python scripts/ab_env.py --m $M --n $N --k $K --strategy stream_k --set SKB200_COOP=0 --set SKB200_COOP=1 --set SKB200_X=1 --rounds 3 --steps 50 --cool 0.3 > gpurun_out/ab_coopauto_$S.json 2>&1
done
timeout 600 python -m paper_2301_03598_b200.sweep --help > gpurun_out/sweep_help.txt 2>&1
timeout 900 python -m paper_2301_03598_b200.sweep --shapes config3 --strategies data_parallel,stream_k:auto,stream_k --out gpurun_out/sweep_c3_coop.csv > gpurun_out/sweep_c3_coop.log 2>&1
timeout 1200 python -m paper_2301_03598_b200.sweep --shapes corpus --count 1000 --strategies data_parallel,stream_k:auto --out gpurun_out/sweep_corpus1000_coop.csv > gpurun_out/sweep_corpus1000_coop.log 2>&1
