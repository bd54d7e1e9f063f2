#!/bin/bash
export MMF_VERBOSE=1
for c in 4 5 3; do
timeout 300 python tools/prof.py --config $c --sweeps 3 --time --opt kernels=6 2>&1 | grep -v "^\[mmf\] order" | tail -3
done
timeout 300 python tools/prof.py --config 4 --sweeps 1 --opt kernels=6 2>&1 | grep "order cand" | sort -t' ' -k14 -n | head -8
