#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "config_parity or pipelined or invariants or tight or tiny" > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt.log
for L in 256 1024; do
  timeout 300 python tools/prof.py --config 4 --L $L --sweeps 3 --time 2>&1 | tail -1
done
