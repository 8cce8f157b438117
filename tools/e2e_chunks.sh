#!/bin/bash
# e2e time of the host-buffer product vs the number of row chunks (KGP_HOST_CHUNKS)
for c in 1 2 3 4; do
  KGP_HOST_CHUNKS=$c timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --skip-nlml 2>/dev/null \
    | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('chunks', $c, 'e2e ms', round(d['e2e']['ms_per_step'], 3))"
done
