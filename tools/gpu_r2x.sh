#!/bin/bash
for c in 4 5; do
  timeout 120 python tools/prof.py --config $c --sweeps 3 --time 2>&1 | grep -E "fwd_fused|rror" | tr '\n' ' '; echo " [cfg $c]"
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "config_parity or pipelined or invariants or tight" > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt.log
