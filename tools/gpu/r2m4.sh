# round-2 multi-GPU: bench at N = 1, 2, 4 (headline, no sweep) + sharded parity check
set -x
mkdir -p gpurun_out
nvidia-smi -L
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python bench.py --steps 5 --warmup 2 --no-latency --no-cpu-baseline --no-sweep > gpurun_out/r2m_n1.json 2> gpurun_out/r2m_n1.err
timeout 900 $TR --nproc-per-node 2 --master-port 29521 bench.py --gpus 2 --steps 5 --warmup 2 --no-latency --no-cpu-baseline > gpurun_out/r2m_n2.json 2> gpurun_out/r2m_n2.err
timeout 900 $TR --nproc-per-node 4 --master-port 29522 bench.py --gpus 4 --steps 5 --warmup 2 --no-latency --no-cpu-baseline > gpurun_out/r2m_n4.json 2> gpurun_out/r2m_n4.err
timeout 900 $TR --nproc-per-node 4 --master-port 29523 tools/check_sharded.py > gpurun_out/r2m_check4.log 2>&1; tail -5 gpurun_out/r2m_check4.log
timeout 900 $TR --nproc-per-node 2 --master-port 29524 tools/check_sharded.py > gpurun_out/r2m_check2.log 2>&1; tail -5 gpurun_out/r2m_check2.log
for n in 1 2 4; do python -c "
import json,sys; d=json.load(open('gpurun_out/r2m_n$n.json')); print($n, '%.3e'%d['value'], round(d['ms_per_step'],1), '%.3e'%d['e2e']['value'], d['schedules_ms']['level_by_level'])"; done
tail -3 gpurun_out/r2m_n4.err
