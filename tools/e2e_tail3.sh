#!/bin/bash
# e2e time vs the geometric row chunking of the output copies (KGP_HOST_CHUNKS, KGP_HOST_RRATIO)
run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --skip-nlml --skip-secondary 2>/dev/null \
    | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', 'e2e ms', round(d['e2e']['ms_per_step'], 3), 'step ms', round(d['ms_per_step'], 3))"; }
KGP_HOST_CHUNKS=3 KGP_HOST_RRATIO=0 run "rows3 tail35 (old)"
for c in 3 4 5 6 8; do for q in 40 50 65; do KGP_HOST_CHUNKS=$c KGP_HOST_RRATIO=$q run "rows$c q$q"; done; done
KGP_HOST_CHUNKS=4 KGP_HOST_RRATIO=50 run "rows4 q50 again"
