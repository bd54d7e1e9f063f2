#!/bin/bash
python tools/prof.py --config 4 --sweeps 1 > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fwd_pipe -s 230 -c 1 -o gpurun_out/ncu_fwd_cur \
    python tools/prof.py --config 4 --sweeps 1 > gpurun_out/ncu_fcur.log 2>&1; echo "ncu rc=$?"
