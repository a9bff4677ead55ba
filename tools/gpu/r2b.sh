# round-2: GPU tests, then the new bench (4096x1024 headline, sweep, latencies, CPU legs), reference arm
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2b_pytest.log 2>&1; tail -3 gpurun_out/r2b_pytest.log
/usr/bin/time -v true 2>/dev/null
start=$(date +%s)
timeout 1500 python bench.py --steps 2 --warmup 1 > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
echo "bench rc=$? wall=$(( $(date +%s) - start ))s"
start=$(date +%s)
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2b_ref.json 2> gpurun_out/r2b_ref.err
echo "ref rc=$? wall=$(( $(date +%s) - start ))s"
tail -c 3000 gpurun_out/r2b_bench.json; tail -n 5 gpurun_out/r2b_bench.err; cat gpurun_out/r2b_ref.json; tail -n 5 gpurun_out/r2b_ref.err
