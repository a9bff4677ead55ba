# list-kernel residency sweep (DP_LIST_MIN_BLOCKS 6 / 8 / 10 / 12) on the headline
for v in base list6 list10 list12; do
  if [ $v = base ]; then L=""; else L="PIPECUT_B200_LIB=build/var/$v/libpipecut_b200.so"; fi
  echo "== $v"; env $L timeout 600 python tools/profile_dp.py --nb 4096 --D 256 --reps 3 2>&1 | tail -2
  env $L timeout 600 python tools/profile_dp.py --nb 4096 --D 1024 --reps 1 2>&1 | tail -1
done > gpurun_out/r2bi.log 2>&1
