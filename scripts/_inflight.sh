for k in 2 3 4 6; do
python bench.py --steps 20 --warmup 5 --inflight $k 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=1 inflight=$k', d['value'], d['ms_per_step'])"
done
for n in 4; do for k in 4 6 8 4; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 20 --warmup 5 --inflight $k 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=$n inflight=$k', d['value'], d['ms_per_step'])"
done; done
