#!/bin/bash
timeout 400 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "config_parity or pipelined or invariants or tight" > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt.log
for c in 4 5 3; do
  timeout 120 python tools/prof.py --config $c --sweeps 3 --time 2>&1 | tail -1
done
