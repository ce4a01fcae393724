# round-2 HEAD verification + profiles (1 GPU)
set -o pipefail
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2f_gputest.log 2>&1; tail -2 gpurun_out/r2f_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2f_smoke.log
python bench.py > gpurun_out/r2f_bench_n1.json 2> gpurun_out/r2f_bench_n1.err; tail -c 300 gpurun_out/r2f_bench_n1.json
python bench.py --impl reference > gpurun_out/r2f_ref_n1.json 2> gpurun_out/r2f_ref_n1.err; tail -c 300 gpurun_out/r2f_ref_n1.json
python bench.py --steps 2 --warmup 3 --no-gpt --no-e2e --no-cpu-baseline --no-levels > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 900 --csv --log-file gpurun_out/r2f_ncu_launches_n1.csv python bench.py --steps 2 --warmup 3 --no-gpt --no-e2e --no-cpu-baseline --no-levels > gpurun_out/r2f_ncu_bench.log 2>&1; echo "launches rc=$?"
python scripts/prof_fused.py --reps 1 > /dev/null 2>&1 && ncu --set full --import-source on --clock-control none -k regex:quantize_tma32 -c 2 -o gpurun_out/r2f_ncu_fused python scripts/prof_fused.py --reps 1 > gpurun_out/r2f_ncu_fused.log 2>&1; echo "full rc=$?"
