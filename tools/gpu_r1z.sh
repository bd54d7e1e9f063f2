#!/bin/bash
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "config_parity or pipelined or invariants or tight" > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt.log
for L in 256 1024; do
for o in "" "--opt dry=1"; do
  timeout 120 python tools/prof.py --config 4 --L $L --sweeps 3 --time $o 2>&1 | tail -1
done; done
