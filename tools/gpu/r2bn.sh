# bisect the sporadic form_stage host stalls: pre-k_refine (A), k_refine (B), pinned read-back (C), HEAD
for rep in 1 2; do
for v in A B C HEAD; do
  if [ $v = HEAD ]; then d=.; else d=build/wt/$v; fi
  echo "== $v rep $rep"; (cd $d && timeout 600 python tools/lat_probe.py C3 C4)
done; done
