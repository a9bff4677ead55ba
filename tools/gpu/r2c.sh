# round-2: new parity tests (negative times, C5 goldens so far) + per-level costs for schedule (i)
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_negative_times.py tests/test_gpu_c5_golden.py -m gpu -x -q > gpurun_out/r2c_pytest.log 2>&1; tail -15 gpurun_out/r2c_pytest.log
timeout 600 python tools/level_costs.py > gpurun_out/r2c_levels.log 2>&1; cat gpurun_out/r2c_levels.log
