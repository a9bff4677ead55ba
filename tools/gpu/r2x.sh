# round-2 validation + ncu evidence for the final kernel
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --deselect tests/test_gpu_c5_golden.py::test_first_level_grid_complete > gpurun_out/r2x_pytest.log 2>&1; tail -3 gpurun_out/r2x_pytest.log
PIPECUT_B200_BOUND_MIN_VISITS=0 timeout 1500 python -m pytest tests -m gpu -q --deselect tests/test_gpu_c5_golden.py::test_first_level_grid_complete > gpurun_out/r2x_pytest_bound0.log 2>&1; tail -3 gpurun_out/r2x_pytest_bound0.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
B="python bench.py --steps 1 --warmup 0 --no-sweep --no-latency --no-cpu-baseline"
timeout 1200 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,sm__inst_executed_pipe_fp64.sum,smsp__thread_inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --kernel-name regex:k_dp_level --clock-control none --csv --log-file gpurun_out/r2x_dp_inst.csv $B > gpurun_out/r2x_ncu1.log 2>&1; echo ncu1 rc=$?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2x_launches.csv $B > gpurun_out/r2x_ncu2.log 2>&1; echo ncu2 rc=$?
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:k_dp_level_list --launch-skip 40 --launch-count 1 -o gpurun_out/r2x_dp_list40 python tools/profile_dp.py --nb 4096 --D 256 --reps 1 > gpurun_out/r2x_ncu3.log 2>&1; echo ncu3 rc=$?
wc -l gpurun_out/r2x_*.csv
