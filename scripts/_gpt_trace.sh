mkdir -p /tmp/tr
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 scripts/gpt_step.py --model gpt-1.3b --batch 1 --seq 1024 --steps 4 --warmup 3 --modes fsdp,qsdp --trace /tmp/tr/t13 2>&1 | tail -1
python scripts/trace_summary.py /tmp/tr/t13_fsdp.json /tmp/tr/t13_qsdp.json
