#!/bin/bash
# isolate pipeline components of the tcgen05 operator (results are wrong with debug flags set)
for f in 0 1 2 3 4 5 6 7; do echo "KGP_TC_DEBUG=$f"; KGP_TC_DEBUG=$f timeout 120 python tools/tc_variants.py ${N:-32768} | grep -E "k= 32"; done
