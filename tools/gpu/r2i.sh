set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --deselect tests/test_gpu_c5_golden.py::test_first_level_grid_complete > gpurun_out/r2i_pytest.log 2>&1; tail -4 gpurun_out/r2i_pytest.log
PIPECUT_B200_BOUND_MIN_VISITS=0 timeout 1500 python -m pytest tests -m gpu -q --deselect tests/test_gpu_c5_golden.py::test_first_level_grid_complete > gpurun_out/r2i_pytest_bound0.log 2>&1; tail -4 gpurun_out/r2i_pytest_bound0.log
timeout 900 python bench.py --steps 3 --warmup 1 --no-latency --no-cpu-baseline > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err; tail -3 gpurun_out/r2i_bench.err
timeout 900 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,sm__inst_executed_pipe_fp64.sum,smsp__thread_inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --kernel-name regex:k_dp_level --clock-control none --csv --log-file gpurun_out/r2i_dp_inst.csv python bench.py --steps 1 --warmup 0 --no-sweep --no-latency --no-cpu-baseline > gpurun_out/r2i_ncu_bench.log 2>&1; echo ncu rc=$?; wc -l gpurun_out/r2i_dp_inst.csv
