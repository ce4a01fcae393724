python -m pytest tests/test_gpu_comm.py -m gpu -x -q -k "multi_process" 2>&1 | tail -1
for v in 0 1; do for p in 4; do
QSDP_NO_SMALL=$v SWEEP_LOGN=10,12,14 SWEEP_BITS=8 python -m torch.distributed.run --nnodes=1 --nproc-per-node $p --master-addr 127.0.0.1 --master-port 29515 scripts/sweep.py 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('no_small=$v', d['P'], d['collective'], d['n'], d['us'])"
done; done
