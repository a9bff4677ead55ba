for cl in 1 2 4 8 16; do for c in C1 C2 C4; do echo "cluster $cl"; PIPECUT_B200_REFINE_CLUSTER=$cl PIPECUT_B200_BLOCKS_TIMES=1 timeout 300 python tools/time_blocks.py $c; done; done > gpurun_out/r2be_times.log 2>&1
for cl in 1 4 16; do echo "cluster $cl"; PIPECUT_B200_REFINE_CLUSTER=$cl PIPECUT_B200_BLOCKS_TIMES=1 timeout 600 python tools/paper_scale.py 1536; done > gpurun_out/r2be_paper.log 2>&1
timeout 900 python -m pytest tests/test_gpu_blocks.py -m gpu -q -x > gpurun_out/r2be_pytest.log 2>&1; tail -3 gpurun_out/r2be_pytest.log
