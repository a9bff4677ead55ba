set -x
PIPECUT_B200_BOUND_DEBUG=1 timeout 600 python tools/profile_dp.py --nb 4096 --D 256 --reps 1 > gpurun_out/r2j_waves.log 2>&1
grep "chunk\|rep" gpurun_out/r2j_waves.log; grep "U/opt" gpurun_out/r2j_waves.log | grep " MB 1:" | awk '{print $NF}' | sort -n | awk '{a[NR]=$1} END {print "MB1 n", NR, "min", a[1], "p50", a[int(NR*0.5)], "p90", a[int(NR*0.9)], "max", a[NR]}'
PIPECUT_B200_NO_WAVES=1 PIPECUT_B200_BOUND_DEBUG=1 timeout 600 python tools/profile_dp.py --nb 4096 --D 256 --reps 1 > gpurun_out/r2j_nowaves.log 2>&1
grep "chunk\|rep" gpurun_out/r2j_nowaves.log; grep "U/opt" gpurun_out/r2j_nowaves.log | awk '{print $NF}' | sort -n | awk '{a[NR]=$1} END {print "all n", NR, "min", a[1], "p50", a[int(NR*0.5)], "p90", a[int(NR*0.9)], "max", a[NR]}'
PIPECUT_B200_NO_WAVES=1 timeout 600 python tools/profile_dp.py --nb 4096 --D 1024 --reps 1 2>&1 | grep rep
