run() { echo "=== $*"; python bench.py --steps 20 --warmup 3 --no-gpt --no-e2e --no-levels --no-cpu-baseline "$@" > /tmp/b.log 2>&1; tail -1 /tmp/b.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d[\"ms_per_step\"], d[\"value\"], d[\"clocks\"])" || tail -5 /tmp/b.log; }
run
run --inflight 2
run --inflight 3
run --bwd-ag-sms 74 --rs-sms 74
run --bwd-ag-sms 48 --rs-sms 100
run --bwd-ag-sms 100 --rs-sms 48
run --inflight 2 --bwd-ag-sms 74 --rs-sms 74
run --inflight 2 --bwd-ag-sms 48 --rs-sms 100
run --inflight 2 --bwd-ag-sms 32 --rs-sms 116
