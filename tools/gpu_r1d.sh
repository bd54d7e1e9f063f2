#!/bin/bash
python tools/prof.py --config 4 --sweeps 1 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_bwd_head -s 230 -c 1 -o gpurun_out/prof_hbwd4 \
    python tools/prof.py --config 4 --sweeps 1 > gpurun_out/ncu_hbwd.log 2>&1
echo "bwd rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_fwd_head -s 30 -c 1 -o gpurun_out/prof_hfwd4 \
    python tools/prof.py --config 4 --sweeps 1 > gpurun_out/ncu_hfwd.log 2>&1
echo "fwd rc=$?"
