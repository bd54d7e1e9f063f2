#!/bin/bash
for o in "" "--opt fgw=4 --opt fng=1 --opt fnp=2" "--opt fgw=4 --opt fng=1 --opt fnp=3" "--opt fgw=4 --opt fng=2 --opt fnp=2"; do
  MMF_VERBOSE=1 timeout 120 python tools/prof.py --config 4 --sweeps 3 --time $o 2>&1 | grep -E "pipe fwd|fwd_fused|rror" | tr '\n' ' '; echo " [cfg 4 $o]"
done
