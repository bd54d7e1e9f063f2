#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pt_all.log 2>&1; echo "pytest all rc=$?"; tail -2 gpurun_out/pt_all.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench4 rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_c4.json')); print(d['ms_per_step'], '%.3e'%d['value'], d['roofline']['frac'], '%.3e'%d['e2e']['value'], d['e2e']['seconds'], d['kernel_breakdown_ms_per_step'])"
timeout 600 python tools/e2e_breakdown.py --config 4 2>&1 | grep "^rep"
