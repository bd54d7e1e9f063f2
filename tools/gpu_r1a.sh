#!/bin/bash
# round-1 re-entry check: GPU tests, bench line, per-kernel timing, launch list
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo "bench rc=$?"
cat gpurun_out/bench4.json
timeout 300 python tools/prof.py --config 4 --sweeps 3 --time > gpurun_out/prof4.log 2>&1; tail -2 gpurun_out/prof4.log
timeout 300 python tools/prof.py --config 5 --sweeps 3 --time > gpurun_out/prof5.log 2>&1; tail -2 gpurun_out/prof5.log
timeout 300 python tools/prof.py --config 3 --sweeps 3 --time > gpurun_out/prof3.log 2>&1; tail -2 gpurun_out/prof3.log
