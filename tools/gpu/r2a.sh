# round-2 probe: GPU tests after the span-marker/offset changes, then nb=4096 points
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_pytest.log 2>&1; tail -5 gpurun_out/r2a_pytest.log
PIPECUT_B200_LEVELS=1 timeout 600 python bench.py --nb 4096 --D 64 --steps 1 --warmup 1 --no-cpu-baseline --no-latency > gpurun_out/r2a_nb4096_D64.json 2> gpurun_out/r2a_nb4096_D64.err
PIPECUT_B200_LEVELS=1 timeout 900 python bench.py --nb 4096 --D 256 --steps 1 --warmup 1 --no-cpu-baseline --no-latency > gpurun_out/r2a_nb4096_D256.json 2> gpurun_out/r2a_nb4096_D256.err
tail -c 1500 gpurun_out/r2a_*.json; tail -5 gpurun_out/r2a_*.err
