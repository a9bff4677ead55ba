# is the DP's device time sensitive to host load (launch-queue stalls)?
nproc
timeout 600 python tools/profile_dp.py --nb 4096 --D 256 --reps 3 2>&1 | tail -2
pids=""
for i in $(seq 1 $(( $(nproc) * 2 ))); do (timeout 120 python3 -c "while True: pass") & pids="$pids $!"; done
sleep 2
timeout 600 python tools/profile_dp.py --nb 4096 --D 256 --reps 3 2>&1 | tail -2
for p in $pids; do kill $p 2>/dev/null; done
wait
