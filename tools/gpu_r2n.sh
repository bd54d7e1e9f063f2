#!/bin/bash
MMF_VERBOSE=1 timeout 120 python tools/prof.py --config 4 --sweeps 3 --time 2>&1 | grep -E "reuse|pipe fwd|fwd_fused|rror" | head -20
MMF_VERBOSE=1 timeout 120 python tools/prof.py --config 4 --sweeps 3 --time --opt bwd=1 2>&1 | grep -E "fwd_fused|rror"
MMF_VERBOSE=1 timeout 120 python tools/prof.py --config 5 --sweeps 2 --time 2>&1 | grep -E "reuse|fwd_fused|rror" | head -20
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "config_parity or pipelined or invariants or kernel_variants or micro" > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pt.log
