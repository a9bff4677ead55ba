# bound floor 2e8: C1-C4 latencies, parity suite
mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/r2ck_bench.json 2> gpurun_out/r2ck_bench.err; echo bench rc=$?
timeout 900 python tools/lat_probe.py > gpurun_out/r2ck_lat.log 2>&1
PIPECUT_B200_BOUND_MIN_VISITS=2e10 timeout 900 python tools/lat_probe.py > gpurun_out/r2ck_lat_old.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2ck_pytest.log 2>&1; tail -1 gpurun_out/r2ck_pytest.log
