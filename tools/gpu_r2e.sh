#!/bin/bash
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench4 rc=$?"
for c in 5 3; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c$c.json 2>gpurun_out/bench_c$c.err; echo "bench$c rc=$?"; done
timeout 300 python bench.py --config 2 --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_c2.json 2>gpurun_out/bench_c2.err; echo "bench2 rc=$?"
timeout 300 python bench.py --config 2 --prec fp32 --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_c2f.json 2>gpurun_out/bench_c2f.err; echo "bench2f rc=$?"
timeout 300 python bench.py --config 1 --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_c1.json 2>gpurun_out/bench_c1.err; echo "bench1 rc=$?"
for f in gpurun_out/bench_c*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['config']['workload'], d['dtype'], round(d['ms_per_step'],3), '%.3e'%d['value'], round(d['hbm_frac_sweep_model'],3), d['kernel_breakdown_ms_per_step'])"; done
python tools/prof.py --config 4 --sweeps 1 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_bwd_pipe2 -s 230 -c 1 -o gpurun_out/ncu_bwd_r01g \
    python tools/prof.py --config 4 --sweeps 1 > gpurun_out/ncu_pbwd.log 2>&1
echo done
