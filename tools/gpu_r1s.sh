#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_gpu.log | grep -v "^$" | tail -4
for c in 4 5 3; do
timeout 300 python tools/prof.py --config $c --sweeps 3 --time 2>&1 | tail -2
timeout 300 python tools/prof.py --config $c --sweeps 3 --time --opt kernels=6 2>&1 | tail -2
done
python tools/prof.py --config 4 --sweeps 1 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_fwd_pipe -s 5 -c 1 -o gpurun_out/prof_pfwd4d \
    python tools/prof.py --config 4 --sweeps 1 > gpurun_out/ncu_pfwd.log 2>&1
