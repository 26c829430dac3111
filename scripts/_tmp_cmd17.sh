mkdir -p gpurun_out
timeout 400 python scripts/ab_env.py --strategy two_tile_sk_dp --set SKB200_TILE_GROUP=1 --set SKB200_TILE_GROUP=8 --set SKB200_TILE_GROUP=4 --set SKB200_TILE_GROUP=16 --rounds 4 --steps 20 --cool 1 --no-check > gpurun_out/ab_tg_2t.json 2>&1
timeout 400 python scripts/ab_env.py --strategy data_parallel --set SKB200_TILE_GROUP=1 --set SKB200_TILE_GROUP=8 --rounds 3 --steps 20 --cool 1 > gpurun_out/ab_tg_dp.json 2>&1
