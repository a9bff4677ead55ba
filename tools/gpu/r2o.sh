set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_bound.py tests/test_gpu_c5_golden.py -m gpu -q --deselect tests/test_gpu_c5_golden.py::test_first_level_grid_complete > gpurun_out/r2o_pytest.log 2>&1; tail -6 gpurun_out/r2o_pytest.log
for c in C1 C2 C3 C4; do PIPECUT_B200_BLOCKS_TIMES=1 timeout 300 python tools/time_blocks.py $c 2>&1 | tail -12; done > gpurun_out/r2o_blocks.log; cat gpurun_out/r2o_blocks.log | tail -60
