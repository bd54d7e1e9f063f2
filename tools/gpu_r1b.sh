#!/bin/bash
# ncu: launch list of the bench command + full capture of the forward and backward sweep kernels on cfg [4]
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/b_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1300 --csv --log-file gpurun_out/launches_r01.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
python tools/prof.py --config 4 --sweeps 1 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_fwd_wide -s 30 -c 1 -o gpurun_out/prof_fwd4 \
    python tools/prof.py --config 4 --sweeps 1 > gpurun_out/ncu_fwd.log 2>&1
echo "fwd rc=$?"
ncu --set full --clock-control none --import-source on -k regex:k_bwd_wide -s 230 -c 1 -o gpurun_out/prof_bwd4 \
    python tools/prof.py --config 4 --sweeps 1 > gpurun_out/ncu_bwd.log 2>&1
echo "bwd rc=$?"
