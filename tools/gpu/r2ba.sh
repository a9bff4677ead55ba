set -x
timeout 1500 python -m pytest tests/test_gpu_blocks.py tests/test_gpu_acceptance.py tests/test_gpu_cost_tables.py tests/test_gpu_cli.py -m gpu -q -x > gpurun_out/r2ba_pytest.log 2>&1; tail -3 gpurun_out/r2ba_pytest.log
for c in C1 C2 C3 C4; do PIPECUT_B200_BLOCKS_TIMES=1 timeout 300 python tools/time_blocks.py $c 2>&1 | grep -E "refine|gpu" | tail -3; done
for c in C1 C2 C4; do PIPECUT_B200_HOST_REFINE=1 timeout 300 python tools/time_blocks.py $c 2>&1 | grep -E "gpu" | tail -1; done
PIPECUT_B200_BLOCKS_TIMES=1 timeout 600 python tools/paper_scale.py 1536 2>&1 | tail -9
timeout 1800 python -m pytest tests/test_gpu_c5_golden.py -m gpu -q -x > gpurun_out/r2ba_c5.log 2>&1; tail -3 gpurun_out/r2ba_c5.log
