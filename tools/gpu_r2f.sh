#!/bin/bash
# launch list of the bench command (no ncu first, then under ncu), and a full capture of the forward kernel
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/b_plain.json 2>&1; echo "plain rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_r01f.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/b_ncu.log 2>&1; echo "ncu launches rc=$?"
python tools/launch_summary.py gpurun_out/launches_r01f.csv > gpurun_out/launches_r01f.txt 2>&1; head -12 gpurun_out/launches_r01f.txt
python tools/prof.py --config 4 --sweeps 1 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_fwd_pipe -s 230 -c 1 -o gpurun_out/ncu_fwd_r01h \
    python tools/prof.py --config 4 --sweeps 1 > gpurun_out/ncu_pfwd.log 2>&1; echo "ncu fwd rc=$?"
