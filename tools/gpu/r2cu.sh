# non-DP time of a headline batch: before / after the triage-factor commit, same box
for v in prev cur prev cur; do
  if [ $v = prev ]; then d=build/wt/prev; else d=.; fi
  echo "== $v"; (cd $d && timeout 600 python tools/profile_dp.py --nb 4096 --D 256 --reps 3 2>&1 | tail -2)
done
