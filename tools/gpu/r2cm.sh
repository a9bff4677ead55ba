# greedy bound: best of extras-first / last / spread device splits
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_bound.py tests/test_gpu_c5_golden.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/r2cm_pytest.log 2>&1; tail -1 gpurun_out/r2cm_pytest.log
timeout 600 python tools/profile_dp.py --nb 4096 --D 256 --reps 3 2>&1 | tail -2
timeout 900 python tools/profile_dp.py --nb 4096 --D 1024 --reps 1 2>&1 | tail -1
PIPECUT_B200_BOUND_DEBUG=1 timeout 600 python tools/profile_dp.py --nb 4096 --D 256 --reps 1 > gpurun_out/r2cm.log 2>&1
