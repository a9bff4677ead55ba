# list order d-major (pool locality) vs b-major
for v in base dmajor base dmajor; do
  if [ $v = base ]; then L=""; else L="PIPECUT_B200_LIB=build/var/$v/libpipecut_b200.so"; fi
  echo "== $v"; env $L timeout 600 python tools/profile_dp.py --nb 4096 --D 256 --reps 3 2>&1 | tail -2
done > gpurun_out/r2bx.log 2>&1
PIPECUT_B200_LIB=build/var/dmajor/libpipecut_b200.so timeout 900 python tools/profile_dp.py --nb 4096 --D 1024 --reps 1 >> gpurun_out/r2bx.log 2>&1
timeout 900 python tools/profile_dp.py --nb 4096 --D 1024 --reps 1 >> gpurun_out/r2bx.log 2>&1
