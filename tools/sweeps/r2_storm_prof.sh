#!/bin/bash
# Storm profile (2 ranks on cuda:0): 4 MiB ring (held frames overflow into rendezvous) and 64 MiB ring.
exec > gpurun_out/r2_storm_prof.txt 2>&1
echo "== ring 4M (default)"; timeout 300 python tools/storm_profile.py 20000 --no-profile
echo "== ring 64M"; M4D_EAGER_DEVICE_RING=67108864 timeout 300 python tools/storm_profile.py 20000 --no-profile
echo "== proxy off, ring 64M"; M4D_EAGER_PROXY=0 M4D_EAGER_DEVICE_RING=67108864 timeout 300 python tools/storm_profile.py 20000 --no-profile
