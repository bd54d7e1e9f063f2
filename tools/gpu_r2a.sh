#!/bin/bash
python tools/prof.py --config 4 --sweeps 1 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_fwd_pipe -s 5 -c 1 -o gpurun_out/prof_pfwd4e \
    python tools/prof.py --config 4 --sweeps 1 > gpurun_out/ncu_pfwd.log 2>&1
