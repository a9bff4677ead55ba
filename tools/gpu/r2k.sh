set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --deselect tests/test_gpu_c5_golden.py::test_first_level_grid_complete > gpurun_out/r2k_pytest.log 2>&1; tail -4 gpurun_out/r2k_pytest.log
PIPECUT_B200_BOUND_MIN_VISITS=0 timeout 1500 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_c5_golden.py::test_first_level_grid_complete > gpurun_out/r2k_pytest_bound0.log 2>&1; tail -4 gpurun_out/r2k_pytest_bound0.log
PIPECUT_B200_LEVELS=1 timeout 600 python tools/profile_dp.py --nb 4096 --D 256 --reps 2 2>&1 | tail -4
PIPECUT_B200_LEVELS=1 timeout 600 python tools/profile_dp.py --nb 4096 --D 1024 --reps 1 2>&1 | tail -3
