# round-2: objective bound with MB waves -- full GPU suite, timing with/without the bound
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2e_pytest.log 2>&1; tail -5 gpurun_out/r2e_pytest.log
timeout 600 python tools/profile_dp.py --nb 4096 --D 256 --reps 2 2>&1 | tail -2
PIPECUT_B200_NO_BOUND=1 timeout 600 python tools/profile_dp.py --nb 4096 --D 256 --reps 2 2>&1 | tail -2
timeout 600 python tools/profile_dp.py --nb 4096 --D 1024 --reps 1 2>&1 | tail -1
timeout 600 python tools/profile_dp.py --nb 1024 --D 256 --reps 2 2>&1 | tail -1
