python -m pytest tests/test_gpu_comm.py tests/test_gpu_fsdp.py -m gpu -x -q 2>&1 | tail -15
for b in 1 4; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 scripts/gpt_step.py --model gpt-1.3b --batch $b --seq 1024 --steps 8 --warmup 3 --modes nocomm,fsdp,qsdp --out gpurun_out/gpt13b_n4_b$b.json 2>&1 | tail -1
done
