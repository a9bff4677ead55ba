# cudaMemGetInfo cached: C1-C4 latency runs (were sporadically +5..+90 ms)
for rep in 1 2; do timeout 900 python tools/lat_probe.py; done > gpurun_out/r2bu.log 2>&1
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_cost_tables.py -m gpu -q -x > gpurun_out/r2bu_pytest.log 2>&1; tail -1 gpurun_out/r2bu_pytest.log
