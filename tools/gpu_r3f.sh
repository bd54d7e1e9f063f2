#!/bin/bash
timeout 600 python tools/e2e_breakdown.py --config 4 2>&1 | grep "^rep\|rror"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pt_all.log 2>&1; echo "pytest all rc=$?"; tail -2 gpurun_out/pt_all.log
