#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pytest_gpu.log | grep -v "^$" | tail -3
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r01d.json 2> gpurun_out/bench_r01d.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_r01d.json')); print(d['value'], d['ms_per_step'], d['hbm_frac_sweep_model'], d['roofline']['frac'], d['kernel_breakdown_ms_per_step'], d['clocks'])"
python tools/prof.py --config 4 --sweeps 1 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_fwd_pipe -s 5 -c 1 -o gpurun_out/ncu_fwd_r01f \
    python tools/prof.py --config 4 --sweeps 1 > gpurun_out/ncu_pfwd.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_bwd_pipe2 -s 230 -c 1 -o gpurun_out/ncu_bwd_r01f \
    python tools/prof.py --config 4 --sweeps 1 > gpurun_out/ncu_pbwd.log 2>&1
echo done
