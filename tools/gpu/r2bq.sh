for v in new old new old; do
  if [ $v = new ]; then L=""; else L="PIPECUT_B200_LIB=build/var/oldgreedy/libpipecut_b200.so"; fi
  echo "== $v"; env $L timeout 600 python tools/sched_probe.py 2>&1 | tail -5
done
