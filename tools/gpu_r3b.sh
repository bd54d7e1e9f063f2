#!/bin/bash
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pt_all.log 2>&1; echo "pytest all rc=$?"; tail -2 gpurun_out/pt_all.log
for c in 4 5; do
timeout 900 python bench.py --config $c --steps 5 --warmup 3 $([ $c != 4 ] && echo --no-cpu) > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; echo "bench$c rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_c$c.json')); print($c, d['ms_per_step'], '%.3e'%d['value'], d['roofline']['frac'], d['kernel_breakdown_ms_per_step'])"
done
