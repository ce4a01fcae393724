python -m pytest tests/test_gpu_kernels.py tests/test_gpu_comm.py -m gpu -x -q 2>&1 | tail -1
for i in 1 2 3; do python bench.py --steps 20 --warmup 5 --no-e2e --no-gpt --no-levels 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=1', d['value'], d['ms_per_step'], d['roofline']['frac_by_kernel'])"; done
