python -m pytest tests/test_gpu_kernels.py tests/test_gpu_protocol.py tests/test_gpu_comm.py -x -q -m gpu -p no:cacheprovider 2>&1 | tail -2
for S in 64 128 256 512 1024 2048 4096; do
python bench.py --model gpt2-350m --wbits 8 --gbits 4 --bucket $S --steps 10 --no-gpt --no-e2e --no-levels --no-cpu-baseline > /tmp/b.json 2>/tmp/b.err || tail -3 /tmp/b.err
tail -1 /tmp/b.json > gpurun_out/bench350_S$S.json
python -c "import json; d=json.load(open('gpurun_out/bench350_S$S.json')); k=d['kernels']; print($S, d['value'], d['ms_per_step'], {n:v['gbs'] for n,v in k.items()}, d['clocks']['sm_mhz'])"
done
