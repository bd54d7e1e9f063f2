#!/bin/bash
export MMF_VERBOSE=1
for L in 256 512 1024; do
  timeout 300 python tools/prof.py --config 4 --L $L --sweeps 3 --time 2>&1 | grep -v "order cand" | tail -2
  timeout 300 python tools/prof.py --config 4 --L $L --sweeps 3 --time --opt dry=1 2>&1 | tail -1
done
