#!/bin/bash
for o in "" "--opt fgw=2 --opt fng=4 --opt fnp=2"; do
  MMF_VERBOSE=1 timeout 120 python tools/prof.py --config 3 --sweeps 3 --time $o 2>&1 | grep -E "pipe fwd|fwd_fused|rror" | tr '\n' ' '; echo " [cfg 3 $o]"
done
