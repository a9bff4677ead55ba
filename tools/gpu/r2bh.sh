# dynamic chunk sharding vs static LPT at N = 2, 4; blocks parity (coarsening merge pairs)
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_blocks.py -m gpu -q -x > gpurun_out/r2bh_blocks.log 2>&1; tail -2 gpurun_out/r2bh_blocks.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
B="bench.py --steps 10 --warmup 3 --no-latency --no-cpu-baseline --no-sweep"
timeout 900 $TR --nproc-per-node 4 --master-port 29542 $B --gpus 4 > gpurun_out/r2bh_n4.json 2> gpurun_out/r2bh_n4.err
PIPECUT_B200_DYNAMIC_SHARDS=0 timeout 900 $TR --nproc-per-node 4 --master-port 29543 $B --gpus 4 > gpurun_out/r2bh_n4_static.json 2> gpurun_out/r2bh_n4_static.err
timeout 900 $TR --nproc-per-node 2 --master-port 29544 $B --gpus 2 > gpurun_out/r2bh_n2.json 2> gpurun_out/r2bh_n2.err
PIPECUT_B200_DYNAMIC_SHARDS=0 timeout 900 $TR --nproc-per-node 2 --master-port 29545 $B --gpus 2 > gpurun_out/r2bh_n2_static.json 2> gpurun_out/r2bh_n2_static.err
timeout 900 $TR --nproc-per-node 4 --master-port 29546 tools/check_sharded.py > gpurun_out/r2bh_check4.log 2>&1; tail -3 gpurun_out/r2bh_check4.log
for f in n2 n2_static n4 n4_static; do tail -1 gpurun_out/r2bh_$f.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); b=d['breakdown_ms']; print('$f', d['n_gpus'], '%.3e'%d['value'], round(d['ms_per_step'],1), '%.3e'%d['e2e']['value'], 'dp', round(b['dp_ms'],1), 'ex', round(b['exchange_ms'],2), 'run', round(b['run_calls_ms'],1))"; done
