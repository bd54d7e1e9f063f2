#!/bin/bash
python tools/prof.py --config 4 --sweeps 1 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_bwd_pipe -s 230 -c 1 -o gpurun_out/prof_pbwd4 \
    python tools/prof.py --config 4 --sweeps 1 > gpurun_out/ncu_pbwd.log 2>&1
echo "bwd rc=$?"
