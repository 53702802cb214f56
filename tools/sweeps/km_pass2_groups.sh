# pass-2 group count ablation (1e8 rows/side, 1 GPU): ncu times of hist2 / pass-2
timeout 300 python -m pytest tests/test_key_merge_gpu.py -q -x --timeout 200 2>&1 | tail -1
for g in 1 2 4 8; do
  echo "groups=$g"
  M4D_PASS2_GROUPS=$g ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pass2|hist2|group_prefix" -c 3 python tools/prof_km.py --steps 1 2>&1 | grep -E "::|duration" | sed 's/(const.*//'
done
