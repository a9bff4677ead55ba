set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_bound.py tests/test_gpu_c5_golden.py -m gpu -q -x --deselect tests/test_gpu_c5_golden.py::test_first_level_grid_complete > gpurun_out/r2p_pytest.log 2>&1; tail -6 gpurun_out/r2p_pytest.log
timeout 600 python tools/profile_dp.py --nb 4096 --D 256 --reps 2 2>&1 | tail -2
timeout 600 python tools/profile_dp.py --nb 4096 --D 1024 --reps 1 2>&1 | tail -1
timeout 600 python tools/profile_dp.py --nb 1024 --D 256 --reps 2 2>&1 | tail -1
