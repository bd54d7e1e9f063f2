#!/bin/bash
# A/B of library builds (paper_2106_14485_b200/libmmf_<name>.so; "base" = libmmf.so): per-kernel ms per sweep.
#   bash tools/ab_lib.sh "4 5 3" base wh100 ...
CFGS=$1; shift
for c in $CFGS; do for n in "$@"; do
  if [ "$n" = base ]; then L=paper_2106_14485_b200/libmmf.so; else L=paper_2106_14485_b200/libmmf_$n.so; fi
  echo -n "cfg$c $n: "; MMF_LIB=$L timeout 300 python tools/prof.py --config $c --sweeps 3 --time 2>&1 | tail -1
done; done
