python -m pytest tests/test_gpu_kernels.py tests/test_gpu_comm.py -m gpu -x -q 2>&1 | tail -1
QSDP_LIB_PATH=$PWD/paper_2302_02390_b200/_variants/cctab.so python -m pytest tests/test_gpu_kernels.py tests/test_gpu_comm.py -m gpu -x -q 2>&1 | tail -1
for v in head tabct cctab head tabct cctab; do
  case $v in head) export QSDP_LIB_PATH=$PWD/paper_2302_02390_b200/_variants/head.so;; tabct) unset QSDP_LIB_PATH;; cctab) export QSDP_LIB_PATH=$PWD/paper_2302_02390_b200/_variants/cctab.so;; esac
  python bench.py --steps 20 --warmup 5 --no-e2e --no-gpt --no-levels 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v N=1', d['value'], d['ms_per_step'], d['kernels']['RS_K2_fused_dequant']['gbs'])"
done
