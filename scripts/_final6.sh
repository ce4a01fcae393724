set -o pipefail
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2h_gputest.log 2>&1; tail -2 gpurun_out/r2h_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2h_smoke.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/r2h_bench_n1.json 2> gpurun_out/r2h_bench_n1.err; tail -1 gpurun_out/r2h_bench_n1.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=1', d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['gpu_launches'])"
for n in 2 4; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n > gpurun_out/r2h_bench_n$n.json 2> gpurun_out/r2h_bench_n$n.err; tail -1 gpurun_out/r2h_bench_n$n.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=$n', d['value'], d['ms_per_step'], d['e2e']['value'])"
done
