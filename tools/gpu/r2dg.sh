# list pops of 2 cells on the final tree
for v in base grab2 base grab2; do
  if [ $v = base ]; then L=""; else L="PIPECUT_B200_LIB=build/var/$v/libpipecut_b200.so"; fi
  echo "== $v"; env $L timeout 600 python tools/profile_dp.py --nb 4096 --D 256 --reps 3 2>&1 | tail -1
done
