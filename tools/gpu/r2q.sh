# round-2: DP occupancy re-sweep on the bounded kernel (launch bounds 7/8/9/10 CTAs per SM)
set -x
for v in default minb7 minb9 minb10 default; do
  if [ $v = default ]; then L=""; else L="build/var/$v/libpipecut_b200.so"; fi
  echo "== $v"
  PIPECUT_B200_LIB=$L timeout 300 python tools/profile_dp.py --nb 4096 --D 256 --reps 2 2>&1 | tail -1
  PIPECUT_B200_LIB=$L timeout 300 python tools/profile_dp.py --nb 1024 --D 256 --reps 2 2>&1 | tail -1
done
