# tile-scatter CTA size ablation (1e8 rows/side, 1 GPU): ncu time of pass-1 kernels + step digest
timeout 300 python -m pytest tests/test_key_merge_gpu.py -q -x --timeout 200 2>&1 | tail -1
for t in 256 512 1024; do
  echo "threads=$t"
  M4D_TILE_THREADS=$t ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tile_scatter|hist2|pass2" -c 3 python tools/prof_km.py --steps 1 2>&1 | grep -E "::|duration|^\(" | sed 's/(const.*//'
done
