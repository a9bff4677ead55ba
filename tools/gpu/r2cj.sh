# bound size floor re-swept with the -inf bound for calls without a greedy plan
for pt in "256 64" "256 256" "256 1024" "1024 8" "1024 64" "64 64" "64 256" "4096 8"; do
  set -- $pt
  for f in 2e10 0; do
    echo "== nb $1 D $2 floor $f"; PIPECUT_B200_BOUND_MIN_VISITS=$f timeout 600 python tools/profile_dp.py --nb $1 --D $2 --reps 4 2>&1 | tail -1
  done
done > gpurun_out/r2cj.log 2>&1
