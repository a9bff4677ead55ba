set -x
mkdir -p gpurun_out
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name regex:k_dp_level --launch-skip 20 --launch-count 1 -o gpurun_out/r2l_dp_level20 python tools/profile_dp.py --nb 4096 --D 256 --reps 1 > gpurun_out/r2l_ncu.log 2>&1; echo rc=$?; tail -3 gpurun_out/r2l_ncu.log
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name regex:k_dp_level --launch-skip 150 --launch-count 1 -o gpurun_out/r2l_dp_level150 python tools/profile_dp.py --nb 4096 --D 256 --reps 1 > gpurun_out/r2l_ncu2.log 2>&1; echo rc=$?
ls -la gpurun_out/*.ncu-rep
