set -x
for v in grab1 grab2 grab4 grab1 grab2; do
  L="build/var/$v/libpipecut_b200.so"
  echo "== $v"
  PIPECUT_B200_LIB=$L timeout 300 python tools/profile_dp.py --nb 4096 --D 256 --reps 2 2>&1 | tail -1
  PIPECUT_B200_LIB=$L timeout 300 python tools/profile_dp.py --nb 4096 --D 1024 --reps 1 2>&1 | tail -1
done
