#!/bin/bash
for o in "--opt copy=1" "--opt copy=1 --opt dry=1" ""; do
  timeout 300 python tools/prof.py --config 4 --sweeps 3 --time $o 2>&1 | tail -2
done
for o in "--opt copy=1" ""; do
  timeout 300 python tools/prof.py --config 5 --sweeps 3 --time $o 2>&1 | tail -2
  timeout 300 python tools/prof.py --config 3 --sweeps 3 --time $o 2>&1 | tail -2
done
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "pipelined or config_parity or variants" > gpurun_out/pt.log 2>&1; tail -2 gpurun_out/pt.log
