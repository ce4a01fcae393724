# P=4: parity on 4 GPUs with the in-tree lib, then sweep + bench A/B base vs new
python -m pytest tests/test_gpu_comm.py -m gpu -x -q -k "multi_gpu" 2>&1 | tail -3
export SWEEP_LOGN=18,22,26,28 SWEEP_BITS=8
for v in base new base new; do
  if [ $v = base ]; then export QSDP_LIB_PATH=$PWD/paper_2302_02390_b200/_variants/base.so; else unset QSDP_LIB_PATH; fi
  echo "=== $v"
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 scripts/sweep.py 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['collective'], d['n'], d['us'], d['eff_gbs'], d['frac_of_roofline'])"
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 --steps 20 --warmup 5 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['ms_per_step'])"
done
