# which calls of the headline batch run without a bound, and how tight the bound is
mkdir -p gpurun_out
PIPECUT_B200_BOUND_DEBUG=1 timeout 600 python tools/profile_dp.py --nb 4096 --D 256 --reps 1 > gpurun_out/r2cf.log 2>&1
