set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --deselect tests/test_gpu_c5_golden.py::test_first_level_grid_complete > gpurun_out/r2ab_pytest.log 2>&1; tail -3 gpurun_out/r2ab_pytest.log
grep -E "FAIL|Error" gpurun_out/r2ab_pytest.log | head -10
timeout 300 python tools/profile_dp.py --nb 4096 --D 256 --reps 2 2>&1 | tail -1
timeout 300 python tools/profile_dp.py --nb 4096 --D 1024 --reps 1 2>&1 | tail -1
