#!/bin/bash
export MMF_VERBOSE=1
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "config_parity or pipelined or invariants or variants" > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt.log
for o in "" "--opt wintma=0" "--opt dry=1" ; do
  timeout 120 python tools/prof.py --config 4 --sweeps 3 --time $o 2>&1 | grep -v "order cand" | tail -1
done
timeout 120 python tools/prof.py --config 3 --sweeps 3 --time 2>&1 | grep -v "order cand" | tail -1
