# greedy bound: CTA per call, 8-wide T search (dp.cu) -- parity + timing
timeout 1800 python -m pytest tests/test_gpu_bound.py tests/test_gpu_c5_golden.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/r2bp_pytest.log 2>&1; tail -2 gpurun_out/r2bp_pytest.log
timeout 600 python tools/profile_dp.py --nb 4096 --D 256 --reps 3 > gpurun_out/r2bp_prof.log 2>&1; tail -2 gpurun_out/r2bp_prof.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:"k_greedy_bound|k_span_rows" --csv --log-file gpurun_out/r2bp_launches.csv python bench.py --steps 1 --warmup 0 --no-sweep --no-latency --no-cpu-baseline > /dev/null 2>&1; echo ncu rc=$?
timeout 900 python bench.py --steps 5 --warmup 3 --no-sweep --no-latency --no-cpu-baseline > gpurun_out/r2bp_bench.json 2> gpurun_out/r2bp_bench.err; echo bench rc=$?
