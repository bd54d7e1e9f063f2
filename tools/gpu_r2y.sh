#!/bin/bash
for o in "" "--opt fgw=8 --opt fng=2 --opt fnp=1"; do
  MMF_VERBOSE=1 timeout 120 python tools/prof.py --config 4 --sweeps 3 --time $o 2>&1 | grep -E "pipe fwd|fwd_fused|rror" | tr '\n' ' '; echo " [cfg 4 $o]"
done
