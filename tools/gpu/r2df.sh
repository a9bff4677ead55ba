# multi-GPU with the final tree: bench at N = 1, 2, 4 (headline, no sweep), 4096x1024 on 4, sharded parity
set -x
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python bench.py --steps 10 --warmup 3 --no-latency --no-cpu-baseline --no-sweep > gpurun_out/r2df_n1.json 2> gpurun_out/r2df_n1.err
timeout 900 $TR --nproc-per-node 2 --master-port 29541 bench.py --gpus 2 --steps 10 --warmup 3 --no-latency --no-cpu-baseline > gpurun_out/r2df_n2.json 2> gpurun_out/r2df_n2.err
timeout 900 $TR --nproc-per-node 4 --master-port 29542 bench.py --gpus 4 --steps 10 --warmup 3 --no-latency --no-cpu-baseline > gpurun_out/r2df_n4.json 2> gpurun_out/r2df_n4.err
timeout 900 $TR --nproc-per-node 4 --master-port 29543 bench.py --gpus 4 --nb 4096 --D 1024 --steps 3 --warmup 1 --no-latency --no-cpu-baseline > gpurun_out/r2df_n4_D1024.json 2> gpurun_out/r2df_n4_D1024.err
timeout 900 $TR --nproc-per-node 4 --master-port 29544 tools/check_sharded.py > gpurun_out/r2df_check4.log 2>&1; tail -3 gpurun_out/r2df_check4.log
for f in n1 n2 n4 n4_D1024; do tail -1 gpurun_out/r2df_$f.json | python -c "
import json,sys; d=json.loads(sys.stdin.read()); b=d['breakdown_ms']; print('$f', d['n_gpus'], '%.3e'%d['value'], round(d['ms_per_step'],1), '%.3e'%d['e2e']['value'], 'lvl', round(d['schedules_ms']['level_by_level'],1), 'dp', round(b['dp_ms'],1), 'ex', round(b['exchange_ms'],2))"; done
