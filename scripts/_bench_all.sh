python -m pytest tests/test_gpu_comm.py tests/test_gpu_fsdp.py -m gpu -x -q 2>&1 | tail -2
for n in 4 2; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n > gpurun_out/bench_n$n.json 2> gpurun_out/bench_n$n.err; tail -1 gpurun_out/bench_n$n.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=$n', d['value'], d['ms_per_step'], d['e2e']['value'])"
done
