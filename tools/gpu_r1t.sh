#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_gpu.log | grep -v "^$" | tail -4
MMF_KERNELS=5 timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu5.log 2>&1; echo "pytest k5 rc=$?"; tail -2 gpurun_out/pytest_gpu5.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r01b.json 2> gpurun_out/bench_r01b.err; echo "bench rc=$?"
cat gpurun_out/bench_r01b.json
for c in 5 3 2; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c$c.json 2>gpurun_out/bench_c$c.err; tail -c 700 gpurun_out/bench_c$c.json; echo; done
