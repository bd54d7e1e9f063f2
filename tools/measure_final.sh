#!/bin/bash
# Round-2 final measurement pass (one gpurun call): bench lines for every config, the ncu launch list of the bench command,
# one `ncu --set full` capture of the forward and backward kernels of [4] and of the forward of [5] and [3],
# the schedule comparison on [4] and the scaling floor.  Output: gpurun_out/r02f/ (summaries copied to profiles/r02_final).
O=gpurun_out/r02f; R=/tmp/r02freps; mkdir -p $O $R
python bench.py > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo "bench cfg4 rc=$?"
python bench.py --config 5 --steps 5 > $O/bench_cfg5.json 2> $O/bench_cfg5.err; echo "bench cfg5 rc=$?"
python bench.py --config 3 --steps 5 > $O/bench_cfg3.json 2> $O/bench_cfg3.err; echo "bench cfg3 rc=$?"
python bench.py --config 2 --prec fp64 --steps 10 > $O/bench_cfg2_fp64.json 2> $O/bench_cfg2_fp64.err; echo "bench cfg2 rc=$?"
python bench.py --config 2 --prec fp32 --steps 10 > $O/bench_cfg2_fp32.json 2> $O/bench_cfg2_fp32.err
python bench.py --config 1 --steps 20 > $O/bench_cfg1.json 2> $O/bench_cfg1.err; echo "bench cfg1 rc=$?"
python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_cfg4_reference.json 2> $O/bench_ref.err; echo "ref rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file $O/launches_cfg4.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > $O/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
python tools/launch_summary.py $O/launches_cfg4.csv > $O/launches_cfg4.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_fwd_pipe -s 20 -c 1 -o $R/fwd_cfg4 \
  python tools/prof.py --config 4 --sweeps 1 > $O/ncu_fwd.log 2>&1; echo "ncu fwd rc=$?"
ncu --set full --import-source on --clock-control none -k regex:k_bwd_pipe2 -s 20 -c 1 -o $R/bwd_cfg4 \
  python tools/prof.py --config 4 --sweeps 1 > $O/ncu_bwd.log 2>&1; echo "ncu bwd rc=$?"
ncu --set full --import-source on --clock-control none -k regex:k_fwd_wide -s 20 -c 1 -o $R/fwd_cfg5 \
  python tools/prof.py --config 5 --sweeps 1 > $O/ncu_fwd5.log 2>&1; echo "ncu fwd5 rc=$?"
ncu --set full --import-source on --clock-control none -k regex:k_bwd_tile2 -s 20 -c 1 -o $R/bwd_cfg5 \
  python tools/prof.py --config 5 --sweeps 1 > $O/ncu_bwd5.log 2>&1; echo "ncu bwd5 rc=$?"
ncu --set full --import-source on --clock-control none -k regex:k_fwd_pipe -s 20 -c 1 -o $R/fwd_cfg3 \
  python tools/prof.py --config 3 --sweeps 1 > $O/ncu_fwd3.log 2>&1; echo "ncu fwd3 rc=$?"
ncu --set full --import-source on --clock-control none -k regex:k_bwd_tile2 -s 20 -c 1 -o $R/bwd_cfg3 \
  python tools/prof.py --config 3 --sweeps 1 > $O/ncu_bwd3.log 2>&1; echo "ncu bwd3 rc=$?"
for r in fwd_cfg4 bwd_cfg4 fwd_cfg5 bwd_cfg5 fwd_cfg3 bwd_cfg3; do python tools/ncu_summary.py $R/$r.ncu-rep > $O/ncu_$r.txt 2>&1; done
python tools/ncu_stalls.py $R/fwd_cfg4.ncu-rep > $O/ncu_fwd_cfg4_stalls.txt 2>&1
python tools/make_traffic.py $O > /dev/null 2>&1; echo "traffic rc=$?"
python tools/schedule_compare.py --config 4 --sweeps 30 > $O/schedule_cfg4.json 2> $O/schedule.err; echo "schedule rc=$?"
python tools/scaling_floor.py --out $O/scaling_floor_cfg4.json > /dev/null 2> $O/scaling.err; echo "scaling rc=$?"
python tools/scaling_floor.py --config 5 --sweeps 3 --out $O/scaling_floor_cfg5.json > /dev/null 2> $O/scaling5.err; echo "scaling5 rc=$?"
python tools/e2e_breakdown.py --config 4 --sweeps 10 > $O/e2e_breakdown_cfg4.txt 2>&1; echo "e2e rc=$?"
ls -la $O; du -sh $O
