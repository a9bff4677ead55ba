# triage: level factor table, CTA call cache, early-exit emptiness (dp.cu): parity suites + timing
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2cs_pytest.log 2>&1; tail -1 gpurun_out/r2cs_pytest.log
PIPECUT_B200_BOUND_MIN_VISITS=0 timeout 2400 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_c5_golden.py::test_first_level_grid_complete --deselect tests/test_bench_contract.py::test_gpu_arm_line > gpurun_out/r2cs_pytest_bound0.log 2>&1; tail -1 gpurun_out/r2cs_pytest_bound0.log
timeout 600 python tools/profile_dp.py --nb 4096 --D 256 --reps 3 2>&1 | tail -2
timeout 900 python tools/profile_dp.py --nb 4096 --D 1024 --reps 1 2>&1 | tail -1
timeout 600 python tools/sched_probe.py 2>&1 | tail -3
