#!/bin/bash
# e2e time of the host-buffer product vs the size of the last row chunk (KGP_HOST_TAIL, % of an even share)
for c in ${CHUNKS:-2 3}; do for t in ${TAILS:-100 70 50 35}; do
  KGP_HOST_CHUNKS=$c KGP_HOST_TAIL=$t timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --skip-nlml 2>/dev/null \
    | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chunks', $c, 'tail', $t, 'e2e ms', round(d['e2e']['ms_per_step'], 3))"
done; done
