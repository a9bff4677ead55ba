# host waits: blocking (driver) vs spin-polling, sporadic form_stage stalls
for rep in 1 2; do
for v in block spin; do
  echo "== $v rep $rep"; PIPECUT_B200_SYNC=$v timeout 600 python tools/lat_probe.py
done; done
