#!/bin/bash
# e2e time of the host-buffer product vs the input (column) chunking: KGP_HOST_ZCHUNKS chunks whose
# sizes grow by KGP_HOST_ZRATIO
run() { timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --skip-nlml --skip-secondary 2>/dev/null \
    | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', 'e2e ms', round(d['e2e']['ms_per_step'], 3), 'step ms', round(d['ms_per_step'], 3))"; }
KGP_HOST_ZCHUNKS=1 run "z1"
KGP_HOST_ZCHUNKS=2 KGP_HOST_ZRATIO=1 run "z2 r1"
for z in 2 3 4; do for r in 2 3 4; do KGP_HOST_ZCHUNKS=$z KGP_HOST_ZRATIO=$r run "z$z r$r"; done; done
