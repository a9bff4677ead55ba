# re-tie the instruction profile to dp.cu (comment-only change) + driver-like bench
set -x
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 0 --no-sweep --no-latency --no-cpu-baseline"
timeout 1200 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,sm__inst_executed_pipe_fp64.sum,smsp__thread_inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum --kernel-name regex:k_dp_level --clock-control none --csv --log-file gpurun_out/r2cp_dp_inst.csv $B > gpurun_out/r2cp_ncu1.log 2>&1; echo ncu1 rc=$?
python tools/ncu_inst_summary.py gpurun_out/r2cp_dp_inst.csv 4096 256 256 > gpurun_out/r2cp_dp_level_profile.json && cp gpurun_out/r2cp_dp_level_profile.json profiles/dp_level_profile.json
timeout 1700 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2cp_bench.json 2> gpurun_out/r2cp_bench.err; echo bench rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
