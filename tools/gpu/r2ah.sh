set -x
timeout 1500 python -m pytest tests -m gpu -q --deselect tests/test_gpu_c5_golden.py::test_first_level_grid_complete > gpurun_out/r2ah_pytest.log 2>&1; tail -2 gpurun_out/r2ah_pytest.log
PIPECUT_B200_BOUND_MIN_VISITS=0 timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_acceptance.py tests/test_gpu_bound.py tests/test_gpu_c5_golden.py -m gpu -q --deselect tests/test_gpu_c5_golden.py::test_first_level_grid_complete > gpurun_out/r2ah_pytest_b0.log 2>&1; tail -2 gpurun_out/r2ah_pytest_b0.log
timeout 300 python tools/profile_dp.py --nb 4096 --D 256 --reps 2 2>&1 | tail -1
timeout 300 python tools/profile_dp.py --nb 4096 --D 1024 --reps 1 2>&1 | tail -1
timeout 300 python tools/profile_dp.py --nb 1024 --D 256 --reps 2 2>&1 | tail -1
