#!/bin/bash
MMF_LIB=paper_2106_14485_b200/libmmf_pair.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "pipelined or config_parity or hub or large_ratio" 2>&1 | tail -3
for lib in libmmf.so libmmf_pair.so; do
  MMF_LIB=paper_2106_14485_b200/$lib timeout 300 python tools/prof.py --config 4 --sweeps 3 --time 2>&1 | grep -E "fwd_fused|rror" | tr '\n' ' '; echo " [$lib cfg 4]"
done
