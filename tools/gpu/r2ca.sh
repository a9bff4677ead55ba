# DP work counters (PC_DP_DIAG build): cells, columns, skip searches, chunk lanes on the headline
PIPECUT_B200_DEBUG=1 PIPECUT_B200_LIB=build/var/diag2/libpipecut_b200.so timeout 900 python tools/profile_dp.py --nb 4096 --D 256 --reps 1 > gpurun_out/r2ca2.log 2>&1
