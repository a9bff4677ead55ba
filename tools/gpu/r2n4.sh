# round-2 multi-GPU: LPT weight models at N = 4 (imbalance under the objective bound)
set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for w in device visits cells; do
PIPECUT_B200_SHARD_WEIGHTS=$w PIPECUT_BENCH_VERBOSE=1 timeout 900 $TR --nproc-per-node 4 --master-port 2953${#w} bench.py --gpus 4 --steps 4 --warmup 1 --no-latency --no-cpu-baseline > gpurun_out/r2n_n4_$w.json 2> gpurun_out/r2n_n4_$w.err
tail -1 gpurun_out/r2n_n4_$w.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); b=d['breakdown_ms']; print('$w', '%.3e'%d['value'], round(d['ms_per_step'],1), 'dp', round(b['dp_ms'],1), 'ex', round(b['exchange_ms'],2), 'w', round(b['weights_ms'],1))"
done
