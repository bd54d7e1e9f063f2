#!/bin/bash
# forward consumer-group variants: parity on the pipelined tests, then per-kernel times on [4], [3], [5]
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "config_parity or pipelined or invariants" > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt.log
for o in "" "--opt fgw=4 --opt fng=1" "--opt fgw=8 --opt fng=1"; do
  MMF_VERBOSE=1 timeout 120 python tools/prof.py --config 4 --sweeps 3 --time $o 2>&1 | grep -E "pipe fwd|ms/sweep|fwd_fused"
done
for c in 3 5; do
  for o in "" "--opt fgw=8 --opt fng=1"; do
    MMF_VERBOSE=1 timeout 120 python tools/prof.py --config $c --sweeps 3 --time $o 2>&1 | grep -E "pipe fwd|ms/sweep|fwd_fused"
  done
done
