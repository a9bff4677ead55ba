# round-2 measurement: ncu instruction count of the final kernel -> profile, then the
# driver-like bench and the reference arm
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bound.py tests/test_gpu_c5_golden.py tests/test_gpu_capacity.py -m gpu -q -x --deselect tests/test_gpu_c5_golden.py::test_first_level_grid_complete > gpurun_out/r2ac_pytest.log 2>&1; tail -2 gpurun_out/r2ac_pytest.log
B="python bench.py --steps 1 --warmup 0 --no-sweep --no-latency --no-cpu-baseline"
timeout 1200 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,sm__inst_executed_pipe_fp64.sum,smsp__thread_inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --kernel-name regex:k_dp_level --clock-control none --csv --log-file gpurun_out/r2ac_dp_inst.csv $B > gpurun_out/r2ac_ncu1.log 2>&1; echo ncu1 rc=$?
python tools/ncu_inst_summary.py gpurun_out/r2ac_dp_inst.csv 4096 256 256 > profiles/dp_level_profile.json && cp profiles/dp_level_profile.json gpurun_out/r2ac_dp_level_profile.json
start=$(date +%s)
timeout 1700 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2ac_bench.json 2> gpurun_out/r2ac_bench.err
echo "bench rc=$? wall=$(( $(date +%s) - start ))s"
start=$(date +%s)
timeout 1700 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2ac_ref.json 2> gpurun_out/r2ac_ref.err
echo "ref rc=$? wall=$(( $(date +%s) - start ))s"
tail -3 gpurun_out/r2ac_bench.err
