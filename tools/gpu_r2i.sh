#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "config_parity or pipelined or invariants" > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt.log
for lib in libmmf.so libmmf_owng0.so libmmf_old.so; do
  for o in "--opt fgw=8 --opt fng=1" "" "--opt fgw=4 --opt fng=1"; do
    MMF_LIB=paper_2106_14485_b200/$lib MMF_VERBOSE=1 timeout 120 python tools/prof.py --config 4 --sweeps 3 --time $o 2>&1 | grep -E "pipe fwd|fwd_fused" | tr '\n' ' '; echo " [$lib cfg 4 $o]"
  done
done
