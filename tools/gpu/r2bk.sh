# A/B: suffix bounds handed from k_dp_triage to the list kernel (build/var/lbcache) vs in-tree
for v in base lbcache base lbcache; do
  if [ $v = base ]; then L=""; else L="PIPECUT_B200_LIB=build/var/$v/libpipecut_b200.so"; fi
  echo "== $v"; env $L timeout 600 python tools/profile_dp.py --nb 4096 --D 256 --reps 3 2>&1 | tail -2
done > gpurun_out/r2bk.log 2>&1
PIPECUT_B200_LIB=build/var/lbcache/libpipecut_b200.so timeout 900 python tools/profile_dp.py --nb 4096 --D 1024 --reps 1 >> gpurun_out/r2bk.log 2>&1
PIPECUT_B200_LIB=build/var/lbcache/libpipecut_b200.so timeout 1800 python -m pytest tests/test_gpu_bound.py tests/test_gpu_c5_golden.py tests/test_gpu_parity.py tests/test_gpu_capacity.py -m gpu -q -x > gpurun_out/r2bk_pytest.log 2>&1; tail -2 gpurun_out/r2bk_pytest.log
for i in 1 2; do timeout 900 python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/r2bk_lat$i.json 2> gpurun_out/r2bk_lat$i.err; done
