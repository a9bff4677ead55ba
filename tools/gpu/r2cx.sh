# LPT weights: cells vs visits at N = 2 (headline) and N = 4 (4096 x 1024)
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for w in cells visits; do
  PIPECUT_B200_SHARD_WEIGHTS=$w timeout 900 $TR --nproc-per-node 2 --master-port 2956$((RANDOM % 9)) bench.py --gpus 2 --steps 10 --warmup 3 --no-latency --no-cpu-baseline --no-sweep > gpurun_out/r2cx_n2_$w.json 2> gpurun_out/r2cx_n2_$w.err
  tail -1 gpurun_out/r2cx_n2_$w.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); b=d['breakdown_ms']; print('n2 $w', '%.3e'%d['value'], round(d['ms_per_step'],1), 'dp', round(b['dp_ms'],1), 'ex', round(b['exchange_ms'],2))"
  PIPECUT_B200_SHARD_WEIGHTS=$w timeout 900 $TR --nproc-per-node 4 --master-port 2957$((RANDOM % 9)) bench.py --gpus 4 --nb 4096 --D 1024 --steps 3 --warmup 1 --no-latency --no-cpu-baseline --no-sweep > gpurun_out/r2cx_n4k_$w.json 2> gpurun_out/r2cx_n4k_$w.err
  tail -1 gpurun_out/r2cx_n4k_$w.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); b=d['breakdown_ms']; print('n4 D1024 $w', '%.3e'%d['value'], round(d['ms_per_step'],1), 'dp', round(b['dp_ms'],1), 'ex', round(b['exchange_ms'],2))"
done
