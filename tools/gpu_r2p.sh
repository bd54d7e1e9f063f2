#!/bin/bash
for lib in libmmf.so libmmf_np3.so; do
for c in 4 5; do
  MMF_LIB=paper_2106_14485_b200/$lib MMF_VERBOSE=1 timeout 120 python tools/prof.py --config $c --sweeps 2 --time 2>&1 | grep -E "reuse bwd|fwd_fused|rror" | tr '\n' ' '; echo " [$lib cfg $c]"
done
done
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "config_parity or pipelined or invariants or kernel_variants or micro" > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pt.log
