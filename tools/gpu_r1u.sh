#!/bin/bash
for o in "" "--opt dry=1" "--opt dry=2"; do
  timeout 300 python tools/prof.py --config 4 --sweeps 3 --time $o 2>&1 | tail -1
done
