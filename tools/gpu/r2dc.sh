# deep batches (>= 512 levels) take the 10-CTA list kernel: parity suites, profile, bench, reference arm, 4096x1024 timing
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2dc_pytest.log 2>&1; tail -3 gpurun_out/r2dc_pytest.log
PIPECUT_B200_BOUND_MIN_VISITS=0 timeout 2400 python -m pytest tests -m gpu -q --deselect tests/test_gpu_c5_golden.py::test_first_level_grid_complete > gpurun_out/r2dc_pytest_bound0.log 2>&1; tail -3 gpurun_out/r2dc_pytest_bound0.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
B="python bench.py --steps 1 --warmup 0 --no-sweep --no-latency --no-cpu-baseline"
timeout 1200 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,sm__inst_executed_pipe_fp64.sum,smsp__thread_inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --kernel-name regex:k_dp_level --clock-control none --csv --log-file gpurun_out/r2dc_dp_inst.csv $B > gpurun_out/r2dc_ncu1.log 2>&1; echo ncu1 rc=$?
python tools/ncu_inst_summary.py gpurun_out/r2dc_dp_inst.csv 4096 256 256 > gpurun_out/r2dc_dp_level_profile.json && cp gpurun_out/r2dc_dp_level_profile.json profiles/dp_level_profile.json
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2dc_launches.csv $B > gpurun_out/r2dc_ncu2.log 2>&1; echo ncu2 rc=$?
start=$(date +%s)
timeout 1700 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2dc_bench.json 2> gpurun_out/r2dc_bench.err
echo "bench rc=$? wall=$(( $(date +%s) - start ))s"
start=$(date +%s)
timeout 1700 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2dc_ref.json 2> gpurun_out/r2dc_ref.err
echo "ref rc=$? wall=$(( $(date +%s) - start ))s"
timeout 900 python tools/profile_dp.py --nb 4096 --D 1024 --reps 1 2>&1 | tail -1
