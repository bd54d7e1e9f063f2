#!/bin/bash
# end-of-session refresh: tests, smoke, all bench lines, launch list + ncu of the bench workload's kernels
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pt_all.log 2>&1; echo "pytest all rc=$?"; tail -2 gpurun_out/pt_all.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench4 rc=$?"
for c in 5 3; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c$c.json 2>gpurun_out/bench_c$c.err; echo "bench$c rc=$?"; done
timeout 300 python bench.py --config 2 --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_c2.json 2>gpurun_out/bench_c2.err; echo "bench2 rc=$?"
timeout 300 python bench.py --config 2 --prec fp32 --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_c2f.json 2>gpurun_out/bench_c2f.err; echo "bench2f rc=$?"
timeout 300 python bench.py --config 1 --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_c1.json 2>gpurun_out/bench_c1.err; echo "bench1 rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
for f in gpurun_out/bench_c*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['config']['workload'], d['dtype'], round(d['ms_per_step'],3), '%.3e'%d['value'], round(d['hbm_frac_sweep_model'],3), round(d['roofline']['frac'],3), '%.3e'%d['e2e']['value'], d['kernel_breakdown_ms_per_step'])"; done
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/b_plain.json 2>&1; echo "plain rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file /tmp/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/b_ncu.log 2>&1; echo "ncu launches rc=$?"
python tools/launch_summary.py /tmp/launches.csv > gpurun_out/launches_final.txt 2>&1
python tools/prof.py --config 4 --sweeps 1 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -f -k regex:k_fwd_pipe -s 230 -c 1 -o /tmp/ncu_fwd \
    python tools/prof.py --config 4 --sweeps 1 > gpurun_out/ncu_pfwd.log 2>&1; echo "ncu fwd rc=$?"
python tools/ncu_summary.py /tmp/ncu_fwd.ncu-rep > gpurun_out/ncu_fwd_cfg4_final.txt 2>&1
ncu --set full --clock-control none --import-source on -f -k regex:k_bwd_pipe2 -s 230 -c 1 -o /tmp/ncu_bwd \
    python tools/prof.py --config 4 --sweeps 1 > gpurun_out/ncu_pbwd.log 2>&1; echo "ncu bwd rc=$?"
python tools/ncu_summary.py /tmp/ncu_bwd.ncu-rep > gpurun_out/ncu_bwd_cfg4_final.txt 2>&1
