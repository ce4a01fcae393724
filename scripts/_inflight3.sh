for k in 16 26 16 26; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 --steps 20 --warmup 5 --no-e2e --no-gpt --inflight $k 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=4 inflight=$k', d['value'], d['ms_per_step'])"
done
for k in 16 26; do
python bench.py --steps 20 --warmup 5 --no-e2e --no-gpt --no-levels --inflight $k 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=1 inflight=$k', d['value'], d['ms_per_step'])"
done
