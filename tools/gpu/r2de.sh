# cudaMemGetInfo skipped for batches under a quarter of the last reading: default bench x2, GPU suite
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2de_bench1.json 2> gpurun_out/r2de_bench1.err; echo bench rc=$?
timeout 900 python bench.py --steps 20 --warmup 5 --no-sweep --no-latency --no-cpu-baseline > gpurun_out/r2de_bench2.json 2> gpurun_out/r2de_bench2.err; echo bench rc=$?
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2de_pytest.log 2>&1; tail -1 gpurun_out/r2de_pytest.log
