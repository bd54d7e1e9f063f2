#!/bin/bash
export MMF_VERBOSE=1
MMF_KERNELS=6 timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu6.log 2>&1; echo "pytest k6 rc=$?"; tail -25 gpurun_out/pytest_gpu6.log | grep -v "^$" | tail -4
for c in 4 5 3; do
timeout 300 python tools/prof.py --config $c --sweeps 3 --time --opt kernels=6 2>&1 | grep -v "^\[mmf\] order" | tail -3
done
python tools/prof.py --config 4 --sweeps 1 --opt kernels=6 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_bwd_win -s 230 -c 1 -o gpurun_out/prof_wbwd4c \
    python tools/prof.py --config 4 --sweeps 1 --opt kernels=6 > gpurun_out/ncu_wbwd.log 2>&1
