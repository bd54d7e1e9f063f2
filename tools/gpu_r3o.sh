#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pt_all.log 2>&1; echo "pytest all rc=$?"; tail -2 gpurun_out/pt_all.log
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c3.json 2>gpurun_out/bench_c3.err; echo "bench3 rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_c3.json')); print(d['ms_per_step'], '%.3e'%d['value'], d['roofline']['frac'], d['kernel_breakdown_ms_per_step'])"
