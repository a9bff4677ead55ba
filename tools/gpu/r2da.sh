# final-state check: full GPU suite, smoke, default bench
set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2da_pytest.log 2>&1; tail -2 gpurun_out/r2da_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r2da_bench.json 2> gpurun_out/r2da_bench.err; echo bench rc=$?
