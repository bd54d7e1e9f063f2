#!/bin/bash
export MMF_VERBOSE=1
for c in 4; do
  timeout 300 python tools/prof.py --config $c --sweeps 3 --time --opt kernels=6 2>&1 | tail -3
done
python tools/prof.py --config 4 --sweeps 1 --opt kernels=6 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_bwd_win -s 230 -c 1 -o gpurun_out/prof_wbwd4b \
    python tools/prof.py --config 4 --sweeps 1 --opt kernels=6 > gpurun_out/ncu_wbwd.log 2>&1
