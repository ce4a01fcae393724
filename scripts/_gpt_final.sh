run() { python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 scripts/gpt_step.py --model gpt-1.3b --batch $1 --seq 1024 --steps 12 --warmup 3 --modes $2 --out gpurun_out/g13_b$1_$3.json 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('b=$1', {m: d[m]['ms_per_step'] for m in ('nocomm','fsdp','qsdp') if m in d}, d.get('qsdp_speedup'))"; }
for b in 4 1; do run $b nocomm,fsdp,qsdp a; run $b qsdp,fsdp b; done
