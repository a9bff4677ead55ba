# LPT weights at N = 4 with the final tree: cells (default) / device (feasible pairs) / visits
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
B="bench.py --gpus 4 --steps 10 --warmup 3 --no-latency --no-cpu-baseline --no-sweep"
for w in cells device visits; do
  PIPECUT_B200_SHARD_WEIGHTS=$w timeout 900 $TR --nproc-per-node 4 --master-port 2955$((RANDOM % 9)) $B > gpurun_out/r2cw_$w.json 2> gpurun_out/r2cw_$w.err
  tail -1 gpurun_out/r2cw_$w.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); b=d['breakdown_ms']; print('$w', '%.3e'%d['value'], round(d['ms_per_step'],1), 'dp', round(b['dp_ms'],1), 'ex', round(b['exchange_ms'],2), 'span', round(b['span_ms'],1))"
done
