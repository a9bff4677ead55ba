timeout 900 python -m pytest tests/test_gpu_blocks.py -m gpu -q -x > gpurun_out/r2bd_pytest0.log 2>&1; tail -3 gpurun_out/r2bd_pytest0.log
timeout 1500 python -m pytest tests/test_gpu_acceptance.py tests/test_gpu_cost_tables.py tests/test_gpu_cli.py -m gpu -q -x > gpurun_out/r2bd_pytest.log 2>&1; tail -3 gpurun_out/r2bd_pytest.log
for c in C1 C2 C3 C4; do PIPECUT_B200_BLOCKS_TIMES=1 timeout 300 python tools/time_blocks.py $c; done > gpurun_out/r2bd_times.log 2>&1
for c in C1 C4; do PIPECUT_B200_REFINE_CLUSTER=1 PIPECUT_B200_BLOCKS_TIMES=1 timeout 300 python tools/time_blocks.py $c; done > gpurun_out/r2bd_times_cl1.log 2>&1
PIPECUT_B200_BLOCKS_TIMES=1 timeout 600 python tools/paper_scale.py 1536 > gpurun_out/r2bd_paper.log 2>&1
