#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_gpu.log | grep -v "^$" | tail -3
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r01c.json 2> gpurun_out/bench_r01c.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_r01c.json')); print(d['value'], d['ms_per_step'], d['hbm_frac_sweep_model'], d['roofline']['frac'], d['kernel_breakdown_ms_per_step'])"
