#!/bin/bash
for o in "" ; do
  timeout 120 python tools/prof.py --config 4 --sweeps 3 --time $o 2>&1 | grep -E "fwd_fused|rror" | tr '\n' ' '; echo " [cfg 4 $o]"
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "config_parity or pipelined or tight or kernel_variants" > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt.log
