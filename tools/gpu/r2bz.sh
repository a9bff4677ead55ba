# compute-sanitizer memcheck over every entry point (incl. the device refinement, bounded DP); ncu --set full of the final list kernel
timeout 2400 compute-sanitizer --tool memcheck --leak-check no python tools/sanitize_smoke.py > gpurun_out/r2bz_memcheck.log 2>&1; echo memcheck rc=$?; tail -3 gpurun_out/r2bz_memcheck.log
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name regex:k_dp_level_list --launch-skip 40 --launch-count 1 -o gpurun_out/r2bz_dp_list40 python tools/profile_dp.py --nb 4096 --D 256 --reps 1 > gpurun_out/r2bz_ncu.log 2>&1; echo ncu rc=$?
