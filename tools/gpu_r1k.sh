#!/bin/bash
for o in "--opt order=0" "--opt order=1" "--opt order=0 --opt dry=1" "--opt order=1 --opt dry=1"; do
  timeout 300 python tools/prof.py --config 4 --sweeps 3 --time $o 2>&1 | tail -2
done
for o in "--opt order=0" "--opt order=1"; do
  timeout 300 python tools/prof.py --config 5 --sweeps 3 --time $o 2>&1 | tail -2
  timeout 300 python tools/prof.py --config 3 --sweeps 3 --time $o 2>&1 | tail -2
done
