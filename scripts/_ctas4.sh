python -m pytest tests/test_gpu_comm.py -m gpu -x -q -k "occupancy or single_rank or multi_process" 2>&1 | tail -2
for n in 4 2; do for c in 1 0 1; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 20 --warmup 5 --no-e2e --no-gpt --fwd-ag-ctas $c --bwd-ag-ctas $c 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=$n agctas=$c', d['value'], d['ms_per_step'])"
done; done
