mkdir -p gpurun_out
PIPECUT_B200_LEVELS=1 timeout 600 python tools/profile_dp.py --nb 4096 --D 256 --reps 2 > gpurun_out/r2cz.log 2>&1
