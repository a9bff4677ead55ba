# how much a perfect bound (each call's own optimum) would save over the greedy bound
mkdir -p gpurun_out
PIPECUT_B200_BB_ORACLE=1 timeout 900 python tools/profile_dp.py --nb 4096 --D 256 --reps 1 > gpurun_out/r2ch.log 2>&1
