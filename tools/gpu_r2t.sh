#!/bin/bash
for lib in libmmf.so libmmf_nonorm.so libmmf_nowp.so; do
for c in 4 5; do
  MMF_LIB=paper_2106_14485_b200/$lib timeout 120 python tools/prof.py --config $c --sweeps 3 --time 2>&1 | grep -E "fwd_fused|rror" | tr '\n' ' '; echo " [$lib cfg $c]"
done; done
