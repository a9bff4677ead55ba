# list-kernel residency re-swept on the final tree (DP_LIST_MIN_BLOCKS 6 / 8 / 10)
for v in base list6 list10 base list6 list10; do
  if [ $v = base ]; then L=""; else L="PIPECUT_B200_LIB=build/var/$v/libpipecut_b200.so"; fi
  echo "== $v"; env $L timeout 600 python tools/profile_dp.py --nb 4096 --D 256 --reps 3 2>&1 | tail -1
done > gpurun_out/r2db.log 2>&1
for v in base list10; do
  if [ $v = base ]; then L=""; else L="PIPECUT_B200_LIB=build/var/$v/libpipecut_b200.so"; fi
  echo "== $v 1024"; env $L timeout 900 python tools/profile_dp.py --nb 4096 --D 1024 --reps 1 2>&1 | tail -1
done >> gpurun_out/r2db.log 2>&1
