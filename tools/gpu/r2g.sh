set -x
mkdir -p gpurun_out
PIPECUT_B200_BOUND_DEBUG=1 timeout 600 python tools/profile_dp.py --nb 4096 --D 256 --reps 1 > gpurun_out/r2g_bound.log 2>&1
grep "chunk" gpurun_out/r2g_bound.log; grep "U/opt" gpurun_out/r2g_bound.log | awk '{print $NF}' | sort -n | awk '{a[NR]=$1} END {print "n", NR, "min", a[1], "p10", a[int(NR*0.1)], "p50", a[int(NR*0.5)], "p90", a[int(NR*0.9)], "max", a[NR]}'
timeout 600 python tools/profile_dp.py --nb 4096 --D 256 --reps 2 2>&1 | tail -2
timeout 600 python tools/profile_dp.py --nb 4096 --D 1024 --reps 1 2>&1 | tail -1
timeout 600 python tools/profile_dp.py --nb 1024 --D 256 --reps 2 2>&1 | tail -1
timeout 1200 python -m pytest tests -m gpu -x -q --deselect tests/test_gpu_c5_golden.py::test_first_level_grid_complete > gpurun_out/r2g_pytest.log 2>&1; tail -5 gpurun_out/r2g_pytest.log
