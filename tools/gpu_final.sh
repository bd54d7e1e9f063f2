#!/bin/bash
# final check of the committed state: smoke, the whole GPU suite, the default bench line
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pt_all.log 2>&1; echo "pytest all rc=$?"; tail -2 gpurun_out/pt_all.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/bench_default.json')); print(d['ms_per_step'], '%.3e'%d['value'], d['roofline']['frac'], '%.3e'%d['e2e']['value'], d['clocks'], d['steps'], d['warmup'])"
