# the triage branch for unbounded calls inside bounded batches: partner-plan waves without greedy plans, every batch bounded
mkdir -p gpurun_out
PIPECUT_B200_NO_GREEDY=1 PIPECUT_B200_BOUND_WAVES=1 PIPECUT_B200_BOUND_MIN_VISITS=0 timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_c5_golden.py tests/test_gpu_cost_tables.py tests/test_gpu_fullsize.py tests/test_gpu_negative_times.py -m gpu -q --deselect tests/test_gpu_c5_golden.py::test_first_level_grid_complete > gpurun_out/r2di.log 2>&1; tail -1 gpurun_out/r2di.log
