set -x
PIPECUT_B200_BOUND_DEBUG=1 timeout 600 python tools/profile_dp.py --nb 4096 --D 256 --reps 1 > gpurun_out/r2f_bound.log 2>&1
grep "chunk" gpurun_out/r2f_bound.log; grep "U/opt" gpurun_out/r2f_bound.log | awk '{print $NF}' | sort -n | awk '{a[NR]=$1} END {print "n", NR, "min", a[1], "p10", a[int(NR*0.1)], "p50", a[int(NR*0.5)], "p90", a[int(NR*0.9)], "max", a[NR]}'
grep "U/opt" gpurun_out/r2f_bound.log | head -40
