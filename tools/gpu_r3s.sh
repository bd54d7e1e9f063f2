#!/bin/bash
for o in "" "--opt stripw=4" "--opt stripw=8" "--opt stripw=16" "--opt stripw=32"; do
  timeout 300 python tools/prof.py --config 4 --sweeps 3 --time $o 2>&1 | grep -E "fwd_fused|rror" | tr '\n' ' '; echo " [cfg 4 $o]"
done
