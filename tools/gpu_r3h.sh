#!/bin/bash
for lib in libmmf.so libmmf_nopre.so libmmf.so libmmf_nopre.so; do
  MMF_LIB=paper_2106_14485_b200/$lib timeout 120 python tools/prof.py --config 4 --sweeps 3 --time 2>&1 | grep -E "fwd_fused|rror" | tr '\n' ' '; echo " [$lib cfg 4]"
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "config_parity or pipelined or tight or hub" > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt.log
