set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --deselect tests/test_gpu_c5_golden.py::test_first_level_grid_complete > gpurun_out/r2h_pytest.log 2>&1; tail -8 gpurun_out/r2h_pytest.log
timeout 900 python bench.py --steps 3 --warmup 1 --no-latency --no-cpu-baseline > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err; tail -3 gpurun_out/r2h_bench.err
