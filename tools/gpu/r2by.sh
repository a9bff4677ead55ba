# k_span_rows: block/task/dependency indirection loaded one block ahead -- parity + timing
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2by_pytest.log 2>&1; tail -1 gpurun_out/r2by_pytest.log
timeout 600 python tools/profile_dp.py --nb 4096 --D 256 --reps 3 2>&1 | tail -2
timeout 600 python tools/sched_probe.py 2>&1 | tail -4
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:"k_span_rows" --csv --log-file gpurun_out/r2by_launches.csv python bench.py --steps 1 --warmup 0 --no-sweep --no-latency --no-cpu-baseline > /dev/null 2>&1; echo ncu rc=$?
