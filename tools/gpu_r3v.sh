#!/bin/bash
for o in "" "--opt cpt=8" "--opt cpt=2" "--opt prefetch=1" "--opt kernels=4"; do
  timeout 300 python tools/prof.py --config 5 --sweeps 2 --time $o 2>&1 | grep -E "fwd_fused|rror" | tr '\n' ' '; echo " [cfg 5 $o]"
done
