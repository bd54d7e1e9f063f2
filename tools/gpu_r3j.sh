#!/bin/bash
for c in 2 4; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c$c.json 2>gpurun_out/bench_c$c.err; echo "bench$c rc=$?"
python -c "import json,sys; d=json.load(open('gpurun_out/bench_c$c.json')); print(d['config']['workload'], round(d['ms_per_step'],3), '%.3e'%d['value'], '%.3e'%d['e2e']['value'], d['e2e']['seconds'])"; done
timeout 300 python tools/e2e_breakdown.py --config 2 2>&1 | grep "^rep"
