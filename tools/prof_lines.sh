#!/bin/bash
# ncu --set full of one launch of a kernel (regex $1) on config $2, per-line instruction / stall summary.
#   bash tools/prof_lines.sh k_bwd_pipe2 4 bwd4 [extra prof.py args]
K=$1; C=$2; N=$3; shift 3
mkdir -p gpurun_out/p1
ncu --set full --import-source on --clock-control none -k regex:$K -s 20 -c 1 -o gpurun_out/p1/$N \
  python tools/prof.py --config $C --sweeps 1 "$@" > gpurun_out/p1/ncu_$N.log 2>&1; echo "ncu $N rc=$?"
python tools/ncu_lines.py gpurun_out/p1/$N.ncu-rep 400 > gpurun_out/p1/lines_$N.txt 2>&1
python tools/ncu_summary.py gpurun_out/p1/$N.ncu-rep > gpurun_out/p1/sum_$N.txt 2>&1
