python -m pytest tests/test_gpu_comm.py tests/test_gpu_fsdp.py -m gpu -q -p no:cacheprovider > gpurun_out/r2f_gputest_n4box.log 2>&1; tail -2 gpurun_out/r2f_gputest_n4box.log
for n in 2 4; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $n > gpurun_out/r2f_bench_n$n.json 2> gpurun_out/r2f_bench_n$n.err; tail -1 gpurun_out/r2f_bench_n$n.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=$n', d['value'], d['ms_per_step'], d['e2e']['value'], d.get('gpt'))"
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 4 --trace gpurun_out/r2f_tl_n4.json --steps 5 --warmup 3 --no-e2e --no-gpt > /dev/null 2>&1; echo trace rc=$?
