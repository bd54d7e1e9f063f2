#!/bin/bash
for o in "" "--opt dry=1"; do
  timeout 300 python tools/prof.py --config 4 --sweeps 3 --time $o 2>&1 | tail -2
done
timeout 300 python tools/prof.py --config 5 --sweeps 3 --time --opt dry=1 2>&1 | tail -2
