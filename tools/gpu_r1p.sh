#!/bin/bash
export MMF_VERBOSE=1
timeout 300 python tools/prof.py --config 4 --sweeps 3 --time --opt kernels=6 2>&1 | grep -v "^\[mmf\] order" | tail -3
timeout 300 python tools/prof.py --config 4 --sweeps 1 --opt kernels=6 2>&1 | grep "order cand" | sort -t' ' -k12 -n | head -20
