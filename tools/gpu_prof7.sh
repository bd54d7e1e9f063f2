python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
for o in "" "--opt order=0"; do
  python tools/prof.py --config 4 --sweeps 3 --time $o 2>&1 | tail -2
done
python tools/prof.py --config 5 --sweeps 3 --time 2>&1 | tail -2
python tools/prof.py --config 3 --sweeps 3 --time 2>&1 | tail -2
python tools/prof.py --config 4 --sweeps 1 > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_fwd_wide -s 30 -c 1 -o gpurun_out/prof_fwd6 python tools/prof.py --config 4 --sweeps 1 > gpurun_out/ncu_fwd.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_bwd_wide -s 30 -c 1 -o gpurun_out/prof_bwd6 python tools/prof.py --config 4 --sweeps 1 > gpurun_out/ncu_bwd.log 2>&1
echo done
