QSDP_LIB_PATH=$PWD/paper_2302_02390_b200/_variants/addcc.so python -m pytest tests/test_gpu_kernels.py tests/test_gpu_comm.py tests/test_gpu_shared.py tests/test_gpu_protocol.py -m gpu -x -q 2>&1 | tail -1
for v in base new base new; do
  if [ $v = new ]; then export QSDP_LIB_PATH=$PWD/paper_2302_02390_b200/_variants/addcc.so; else unset QSDP_LIB_PATH; fi
  python bench.py --steps 20 --warmup 5 --no-e2e --no-gpt --no-levels 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['value'], d['ms_per_step'], d['kernels']['RS_K2_fused_dequant']['gbs'], d['kernels_unfused']['K2_quantize_stochastic']['gbs'], d['kernels']['AG_K1_fused_dequant']['gbs'])"
done
