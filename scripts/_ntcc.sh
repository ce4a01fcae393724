for v in head ntcc head ntcc; do
  if [ $v = ntcc ]; then export QSDP_LIB_PATH=$PWD/paper_2302_02390_b200/_variants/ntcc.so; else unset QSDP_LIB_PATH; fi
  python bench.py --steps 20 --warmup 5 --no-e2e --no-gpt --no-levels 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v N=1', d['value'], d['ms_per_step'], d['kernels']['RS_K2_fused_dequant']['gbs'])"
done
