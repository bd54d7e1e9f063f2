#!/bin/bash
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu.log
for c in 4 5 3; do
  timeout 300 python tools/prof.py --config $c --sweeps 3 --time 2>&1 | tail -2
done
python tools/prof.py --config 4 --sweeps 1 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_bwd_pipe -s 230 -c 1 -o gpurun_out/prof_pbwd4e \
    python tools/prof.py --config 4 --sweeps 1 > gpurun_out/ncu_pbwd.log 2>&1
