# list pops of 2 cells: other sweep points
for pt in "4096 1024" "4096 64" "1024 256" "1024 1024"; do
  set -- $pt
  for v in base grab2; do
    if [ $v = base ]; then L=""; else L="PIPECUT_B200_LIB=build/var/$v/libpipecut_b200.so"; fi
    echo "== $v $1 $2"; env $L timeout 900 python tools/profile_dp.py --nb $1 --D $2 --reps 2 2>&1 | tail -1
  done
done
