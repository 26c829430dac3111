mkdir -p gpurun_out
M=gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_ltcfabric_op_read.sum
for KA in 0 1; do for L2 in 2,1,1,2 2,1,1,0 0,0,0,0; do
SKB200_L2_POLICY=$L2 SKB200_K_ALIGN=$KA timeout 200 ncu --cache-control none --metrics $M --clock-control none -k regex:sk_gemm -s 5 -c 1 --csv python bench.py --m 1024 --steps 3 --warmup 5 --no-e2e --no-cpu --no-sweep --strategy stream_k > gpurun_out/ncu_ka${KA}_l2${L2}.csv 2>&1
done; done
