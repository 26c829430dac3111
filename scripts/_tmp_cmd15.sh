mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu6.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu6.log
timeout 300 python scripts/ab_env.py --m 1024 --n 8192 --k 8192 --strategy stream_k --set SKB200_K_ALIGN=1 --set SKB200_K_ALIGN=0 --rounds 3 --steps 50 --cool 0.3 > gpurun_out/ab_skphase.json 2>&1
timeout 300 python scripts/ab_env.py --m 1024 --n 8192 --k 8192 --strategy data_parallel --set SKB200_K_ALIGN=1 --rounds 2 --steps 50 --cool 0.3 > gpurun_out/ab_skphase_dp.json 2>&1
M=gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum
for S in stream_k data_parallel; do
timeout 200 ncu --cache-control none --metrics $M --clock-control none -k regex:sk_gemm -s 5 -c 2 --csv python bench.py --m 1024 --steps 3 --warmup 5 --no-e2e --no-cpu --no-sweep --strategy $S > gpurun_out/ncu_skphase_$S.csv 2>&1
done
