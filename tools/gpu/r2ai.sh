set -x
for v in default ctapop ctapop10 default ctapop; do
  if [ $v = default ]; then L=""; else L="build/var/$v/libpipecut_b200.so"; fi
  echo "== $v"
  PIPECUT_B200_LIB=$L timeout 300 python tools/profile_dp.py --nb 4096 --D 256 --reps 2 2>&1 | tail -1
  PIPECUT_B200_LIB=$L timeout 300 python tools/profile_dp.py --nb 4096 --D 1024 --reps 1 2>&1 | tail -1
done
