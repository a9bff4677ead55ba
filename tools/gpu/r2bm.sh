echo "== default"; timeout 600 python tools/lat_probe.py
echo "== cluster 1"; PIPECUT_B200_REFINE_CLUSTER=1 timeout 600 python tools/lat_probe.py
