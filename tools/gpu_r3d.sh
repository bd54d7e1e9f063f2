#!/bin/bash
timeout 120 python tools/prof.py --config 4 --sweeps 3 --time 2>&1 | grep -E "fwd_fused|rror" | tr '\n' ' '; echo " [cfg 4]"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pt_all.log 2>&1; echo "pytest all rc=$?"; tail -2 gpurun_out/pt_all.log
