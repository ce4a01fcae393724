for S in 64 128 256 512 1024 2048 4096; do
python bench.py --model gpt2-350m --gbits 4 --bucket $S --steps 10 --warmup 3 --no-e2e --no-gpt --no-levels --no-cpu-baseline > gpurun_out/b350_S$S.json 2>/dev/null; tail -1 gpurun_out/b350_S$S.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d.get('kernels',{}); print('S=$S', d['value'], d['ms_per_step'], k.get('RS_K2_fused_dequant',{}).get('gbs'))"
done
