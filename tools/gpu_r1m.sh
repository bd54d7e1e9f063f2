#!/bin/bash
# round-1 checkpoint: bench line (default config [4]), launch list of the same command, ncu full captures
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err; echo "bench rc=$?"
cat gpurun_out/bench_r01.json
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/b_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches_r01.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
python tools/prof.py --config 4 --sweeps 1 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_fwd_pipe -s 5 -c 1 -o gpurun_out/ncu_fwd_r01 \
    python tools/prof.py --config 4 --sweeps 1 > gpurun_out/ncu_fwd.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_bwd_pipe -s 230 -c 1 -o gpurun_out/ncu_bwd_r01 \
    python tools/prof.py --config 4 --sweeps 1 > gpurun_out/ncu_bwd.log 2>&1
echo done
