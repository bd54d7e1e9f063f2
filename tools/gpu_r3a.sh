#!/bin/bash
for lib in libmmf.so libmmf_owng1.so; do
for o in "" "--opt fgw=8 --opt fng=1 --opt fnp=3"; do
  MMF_LIB=paper_2106_14485_b200/$lib MMF_VERBOSE=1 timeout 120 python tools/prof.py --config 4 --sweeps 3 --time $o 2>&1 | grep -E "pipe fwd|fwd_fused|rror" | tr '\n' ' '; echo " [$lib cfg 4 $o]"
done; done
