#!/bin/bash
# A/B of forward-kernel configurations on [4] (per-kernel ms per sweep, plain launches)
for o in "" "--opt fgw=4 --opt fng=2 --opt fnp=2" "--opt fgw=4 --opt fng=3 --opt fnp=1" "--opt fgw=8 --opt fng=1 --opt fnp=3" "--opt fgw=8 --opt fng=2 --opt fnp=1"; do
  timeout 300 python tools/prof.py --config 4 --sweeps 3 --time $o 2>&1 | tail -2
done
