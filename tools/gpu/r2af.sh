set -x
timeout 1500 python -m pytest tests -m gpu -q --deselect tests/test_gpu_c5_golden.py::test_first_level_grid_complete > gpurun_out/r2af_pytest.log 2>&1; tail -2 gpurun_out/r2af_pytest.log
timeout 900 python tools/form_stage_modes.py
