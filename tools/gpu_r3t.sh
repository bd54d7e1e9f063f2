#!/bin/bash
for c in 3; do timeout 300 python tools/e2e_breakdown.py --config $c 2>&1 | grep "^rep"; done
timeout 300 python bench.py --config 2 --prec fp32 --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_c2f.json 2>gpurun_out/bench_c2f.err; echo "bench2f rc=$?"
timeout 300 python bench.py --config 2 --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_c2.json 2>gpurun_out/bench_c2.err; echo "bench2 rc=$?"
for f in gpurun_out/bench_c2f.json gpurun_out/bench_c2.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d['config']['workload'], d['dtype'], round(d['ms_per_step'],3), '%.3e'%d['value'], '%.3e'%d['e2e']['value'], d['kernel_breakdown_ms_per_step'])"; done
