#!/bin/bash
# e2e time vs the row chunking of the output copies (KGP_HOST_CHUNKS, KGP_HOST_TAIL) with the input pipelining on
run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --skip-nlml --skip-secondary 2>/dev/null \
    | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', 'e2e ms', round(d['e2e']['ms_per_step'], 3), 'step ms', round(d['ms_per_step'], 3))"; }
for c in 3 4; do for t in 15 25 35 50; do KGP_HOST_CHUNKS=$c KGP_HOST_TAIL=$t run "rows$c tail$t"; done; done
KGP_HOST_CHUNKS=2 KGP_HOST_TAIL=35 run "rows2 tail35"
