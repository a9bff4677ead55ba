# bench with the device refinement (C1-C4 latency lines)
mkdir -p gpurun_out
start=$(date +%s)
timeout 1700 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2bg_bench.json 2> gpurun_out/r2bg_bench.err
echo "bench rc=$? wall=$(( $(date +%s) - start ))s"
tail -3 gpurun_out/r2bg_bench.err
