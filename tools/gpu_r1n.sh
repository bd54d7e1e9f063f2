#!/bin/bash
MMF_KERNELS=6 timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu6.log 2>&1; echo "pytest k6 rc=$?"; tail -25 gpurun_out/pytest_gpu6.log | grep -v "^$" | tail -15
for c in 4 5 3; do
  timeout 300 python tools/prof.py --config $c --sweeps 3 --time --opt kernels=6 2>&1 | tail -2
done
