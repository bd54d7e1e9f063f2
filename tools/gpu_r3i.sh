#!/bin/bash
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pt_all.log 2>&1; echo "pytest all rc=$?"; tail -2 gpurun_out/pt_all.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench4 rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"; cat gpurun_out/bench_ref.json | head -c 600; echo
for c in 5 3; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c$c.json 2>gpurun_out/bench_c$c.err; echo "bench$c rc=$?"; done
timeout 300 python bench.py --config 2 --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_c2.json 2>gpurun_out/bench_c2.err; echo "bench2 rc=$?"
timeout 300 python bench.py --config 2 --prec fp32 --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_c2f.json 2>gpurun_out/bench_c2f.err; echo "bench2f rc=$?"
timeout 300 python bench.py --config 1 --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_c1.json 2>gpurun_out/bench_c1.err; echo "bench1 rc=$?"
for f in gpurun_out/bench_c*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['config']['workload'], d['dtype'], round(d['ms_per_step'],3), '%.3e'%d['value'], round(d['hbm_frac_sweep_model'],3), round(d['roofline']['frac'],3), '%.3e'%d['e2e']['value'], d['kernel_breakdown_ms_per_step'])"; done
