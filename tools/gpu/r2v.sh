set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_bound.py tests/test_gpu_c5_golden.py tests/test_gpu_fullsize.py -m gpu -q -x --deselect tests/test_gpu_c5_golden.py::test_first_level_grid_complete > gpurun_out/r2v_pytest.log 2>&1; tail -3 gpurun_out/r2v_pytest.log
for v in default list10 list8; do
  if [ $v = default ]; then L=""; else L="build/var/$v/libpipecut_b200.so"; fi
  echo "== $v"
  PIPECUT_B200_LIB=$L timeout 300 python tools/profile_dp.py --nb 4096 --D 256 --reps 2 2>&1 | tail -1
  PIPECUT_B200_LIB=$L timeout 300 python tools/profile_dp.py --nb 4096 --D 1024 --reps 1 2>&1 | tail -1
  PIPECUT_B200_LIB=$L timeout 300 python tools/profile_dp.py --nb 1024 --D 256 --reps 2 2>&1 | tail -1
done
