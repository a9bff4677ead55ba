for c in C1 C2 C3 C4; do PIPECUT_B200_BLOCKS_TIMES=1 timeout 300 python tools/time_blocks.py $c; done > gpurun_out/r2bf_times.log 2>&1
PIPECUT_B200_BLOCKS_TIMES=1 timeout 600 python tools/paper_scale.py 1536 > gpurun_out/r2bf_paper.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2bf_pytest.log 2>&1; tail -3 gpurun_out/r2bf_pytest.log
