# DP work counters (PC_DP_DIAG build) on the final tree: what the listed cells still do
mkdir -p gpurun_out
PIPECUT_B200_DEBUG=1 PIPECUT_B200_LIB=build/var/diag5/libpipecut_b200.so timeout 900 python tools/profile_dp.py --nb 4096 --D 256 --reps 1 > gpurun_out/r2ca5.log 2>&1
