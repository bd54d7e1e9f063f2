#!/bin/bash
# head-flow kernels: GPU parity + timing vs the wide kernels
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
for c in 4 5 3; do
  for o in "" "--opt kernels=3" "--opt cpt=8" "--opt cpt=2"; do
    timeout 300 python tools/prof.py --config $c --sweeps 3 --time $o 2>&1 | tail -2
  done
done
