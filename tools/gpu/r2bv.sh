# final-tree bench (after the cudaMemGetInfo fix) + reference arm
set -x
mkdir -p gpurun_out
start=$(date +%s)
timeout 1700 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2bv_bench.json 2> gpurun_out/r2bv_bench.err
echo "bench rc=$? wall=$(( $(date +%s) - start ))s"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
