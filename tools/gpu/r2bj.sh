# end-of-round validation: full GPU suite, smoke, driver-like bench + reference arm
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2bj_pytest.log 2>&1; tail -3 gpurun_out/r2bj_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2bj_smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/r2bj_smoke.log
start=$(date +%s)
timeout 1700 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2bj_bench.json 2> gpurun_out/r2bj_bench.err
echo "bench rc=$? wall=$(( $(date +%s) - start ))s"
start=$(date +%s)
timeout 1700 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2bj_ref.json 2> gpurun_out/r2bj_ref.err
echo "ref rc=$? wall=$(( $(date +%s) - start ))s"
