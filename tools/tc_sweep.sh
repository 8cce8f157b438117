#!/bin/bash
# tuning sweep of runtime knobs of the tcgen05 operator
for d in 1 0; do for f in 4 8 16; do echo "KGP_TC_DEFER=$d KGP_TC_FLUSH=$f"; KGP_TC_DEFER=$d KGP_TC_FLUSH=$f timeout 120 python tools/tc_variants.py 32768 | grep -E "k= 32"; done; done
