mkdir -p gpurun_out/ab
for S in data_parallel two_tile_sk_dp; do
timeout 600 python scripts/ab_env.py --variant 2smw --strategy $S --rounds 3 \
  --set SKB200_RASTER_ROWS=8 --set SKB200_RASTER_ROWS=4 --set SKB200_RASTER_ROWS=6 \
  --set SKB200_RASTER_ROWS=12 --set SKB200_RASTER_ROWS=16 --set SKB200_RASTER_ROWS=32 > gpurun_out/ab/raster_$S.json 2>&1
done
timeout 600 python scripts/ab_env.py --variant 2smw --strategy data_parallel --rounds 3 \
  --set SKB200_L2_POLICY=2,1,1,2 --set SKB200_L2_POLICY=0,0,0,0 --set SKB200_L2_POLICY=2,2,1,2 \
  --set SKB200_L2_POLICY=1,1,1,1 --set SKB200_L2_POLICY=0,1,1,0 > gpurun_out/ab/l2pol_dp.json 2>&1
