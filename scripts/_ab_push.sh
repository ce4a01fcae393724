# A/B of the bulk-store push (in-tree lib) vs base variant at N=2: parity tests then bench pairs
set -x
python -m pytest tests/test_gpu_comm.py tests/test_gpu_fsdp.py -m gpu -x -q 2>&1 | tail -5
for rep in 1 2; do
for v in base new; do
  if [ $v = base ]; then export QSDP_LIB_PATH=$PWD/paper_2302_02390_b200/_variants/base.so; else unset QSDP_LIB_PATH; fi
  echo "=== $v"
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d.get('e2e',{}).get('value'))"
done; done
unset QSDP_LIB_PATH
