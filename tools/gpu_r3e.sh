#!/bin/bash
# bench (default config) + its launch list + full captures of the two step kernels (summaries made here; the
# reports themselves are too large to bring back together)
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?"
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/b_plain.json 2>&1; echo "plain rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file /tmp/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/b_ncu.log 2>&1; echo "ncu launches rc=$?"
python tools/launch_summary.py /tmp/launches.csv > gpurun_out/launches_r01g.txt 2>&1
python tools/prof.py --config 4 --sweeps 1 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_fwd_pipe -s 230 -c 1 -o /tmp/ncu_fwd \
    python tools/prof.py --config 4 --sweeps 1 > gpurun_out/ncu_pfwd.log 2>&1; echo "ncu fwd rc=$?"
python tools/ncu_summary.py /tmp/ncu_fwd.ncu-rep > gpurun_out/ncu_fwd_cfg4_final.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_bwd_pipe2 -s 230 -c 1 -o /tmp/ncu_bwd \
    python tools/prof.py --config 4 --sweeps 1 > gpurun_out/ncu_pbwd.log 2>&1; echo "ncu bwd rc=$?"
python tools/ncu_summary.py /tmp/ncu_bwd.ncu-rep > gpurun_out/ncu_bwd_cfg4_final.txt 2>&1
cp /tmp/ncu_fwd.ncu-rep gpurun_out/ncu_fwd_r01i.ncu-rep
