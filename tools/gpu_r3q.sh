#!/bin/bash
for c in 4 5 3; do
for o in "" "--opt order=1" "--opt order=4"; do
  timeout 300 python tools/prof.py --config $c --sweeps 3 --time $o 2>&1 | grep -E "fwd_fused|rror" | tr '\n' ' '; echo " [cfg $c $o]"
done; done
