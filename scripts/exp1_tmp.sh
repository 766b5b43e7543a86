# ncu A/B: TILED vs TMA tile (cfg 0, pad 20000, evict normal) on 8192^2 f32, one cold launch each
export DESC_TMA_TILE_EVICT=0 DESC_TMA_TILE_SMEM_PAD=20000
for k in tiled tma_tile; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:transpose_ -s 5 -c 1 \
   -o gpurun_out/prof_ab_$k -f python bench.py --kernel $k --steps 8 --warmup 3 --no-oracle --no-e2e > gpurun_out/ncu_ab_$k.log 2>&1
echo "$k rc=$?"
done
