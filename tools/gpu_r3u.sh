#!/bin/bash
for i in 1 2; do timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c3_$i.json 2>gpurun_out/bench_c3.err; python -c "import json; d=json.load(open('gpurun_out/bench_c3_$i.json')); print(d['ms_per_step'], '%.3e'%d['e2e']['value'], d['e2e']['seconds'])"; done
