#!/bin/bash
run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --skip-nlml --skip-secondary 2>/dev/null \
    | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', 'e2e ms', round(d['e2e']['ms_per_step'], 3), 'step ms', round(d['ms_per_step'], 3))"; }
for rep in 1 2; do
for q in 45 50 55; do KGP_HOST_CHUNKS=3 KGP_HOST_RRATIO=$q run "rows3 q$q"; done
KGP_HOST_CHUNKS=3 KGP_HOST_RRATIO=0 run "rows3 tail35 (old)"
KGP_HOST_CHUNKS=2 KGP_HOST_RRATIO=30 run "rows2 q30"
done
