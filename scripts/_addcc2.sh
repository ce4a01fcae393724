python -m pytest tests/test_gpu_kernels.py tests/test_gpu_comm.py -m gpu -x -q 2>&1 | tail -1
for v in base new base new; do
  if [ $v = base ]; then export QSDP_LIB_PATH=$PWD/paper_2302_02390_b200/_variants/base2.so; else unset QSDP_LIB_PATH; fi
  for n in 4; do
  python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n --steps 20 --warmup 5 --no-e2e --no-gpt 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v N=$n', d['value'], d['ms_per_step'])"
  done
  python bench.py --steps 20 --warmup 5 --no-e2e --no-gpt --no-levels 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v N=1', d['value'], d['ms_per_step'], d['kernels_unfused']['K2_quantize_stochastic']['gbs'])"
done
