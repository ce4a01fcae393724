run() { python bench.py --steps 20 --warmup 5 --no-e2e --no-gpt --no-levels --fwd-ag-ctas $1 --bwd-ag-ctas $2 --rs-priority $3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=1 fwd=$1 bwd=$2 prio=$3', d['value'], d['ms_per_step'])"; }
run 1 1 0; run 1 1 -1; run 1 0 -1; run 1 0 0; run 0 1 -1; run 1 1 -1; run 1 1 0
