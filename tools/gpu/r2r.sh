set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_blocks.py tests/test_gpu_acceptance.py tests/test_gpu_cost_tables.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/r2r_pytest.log 2>&1; tail -4 gpurun_out/r2r_pytest.log
for c in C1 C2 C3 C4; do PIPECUT_B200_BLOCKS_TIMES=1 timeout 300 python tools/time_blocks.py $c 2>&1 | grep -E "refine:|gpu"; done
PIPECUT_B200_BLOCKS_TIMES=1 timeout 600 python tools/paper_scale.py 1536 2>&1 | tail -12
for v in minb10 minb11 minb12; do echo "== $v"; PIPECUT_B200_LIB=build/var/$v/libpipecut_b200.so timeout 300 python tools/profile_dp.py --nb 4096 --D 256 --reps 2 2>&1 | tail -1; done
