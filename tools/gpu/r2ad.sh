set -x
PIPECUT_B200_LIB=build/var/cycles/libpipecut_b200.so timeout 300 python tools/profile_dp.py --nb 4096 --D 256 --reps 1 2> gpurun_out/r2ad_cycles_4096_256.log | tail -1
PIPECUT_B200_LIB=build/var/cycles/libpipecut_b200.so timeout 300 python tools/profile_dp.py --nb 4096 --D 1024 --reps 1 2> gpurun_out/r2ad_cycles_4096_1024.log | tail -1
grep -c cycles gpurun_out/r2ad_cycles_*.log
