#!/bin/bash
# One gpurun call: smoke, the GPU suite (optionally a -k filter in $1), the default bench line.
#   /usr/local/graft/bin/gpurun --timeout 1800 -- 'bash tools/gpu_check.sh [pytest -k expr]'
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
if [ -n "$1" ]; then K=(-k "$1"); else K=(); fi
timeout 1500 python -m pytest tests -m gpu -q -x "${K[@]}" > gpurun_out/pt_all.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/pt_all.log
if [ -z "$NOBENCH" ]; then
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_default.json')); print(d['ms_per_step'], '%.3e'%d['value'], d['roofline']['frac'], '%.3e'%d['e2e']['value'], d['clocks'], d['steps'], d['warmup'])"
fi
