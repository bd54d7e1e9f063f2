#!/bin/bash
for o in "" "--opt dry=2" "--opt dry=3" "--opt dry=1"; do
  timeout 120 python tools/prof.py --config 4 --sweeps 3 --time $o 2>&1 | grep -E "fwd_fused|rror" | tr '\n' ' '; echo " [cfg 4 $o]"
done
