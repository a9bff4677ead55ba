for c in C1 C2 C3 C4; do PIPECUT_B200_BLOCKS_TIMES=1 timeout 300 python tools/time_blocks.py $c; done > gpurun_out/r2bb_times.log 2>&1
for c in C1 C2 C4; do PIPECUT_B200_HOST_REFINE=1 timeout 300 python tools/time_blocks.py $c; done > gpurun_out/r2bb_host.log 2>&1
PIPECUT_B200_BLOCKS_TIMES=1 timeout 600 python tools/paper_scale.py 1536 > gpurun_out/r2bb_paper.log 2>&1
PIPECUT_B200_HOST_REFINE=1 PIPECUT_B200_BLOCKS_TIMES=1 timeout 600 python tools/paper_scale.py 1536 > gpurun_out/r2bb_paper_host.log 2>&1
