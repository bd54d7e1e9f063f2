python tools/prof.py --config 4 --sweeps 1 --opt tile=16 > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_fwd_tile -s 30 -c 1 -o gpurun_out/prof_fwd2 python tools/prof.py --config 4 --sweeps 1 --opt tile=16 > gpurun_out/ncu_fwd.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_bwd_tile -s 30 -c 1 -o gpurun_out/prof_bwd2 python tools/prof.py --config 4 --sweeps 1 --opt tile=16 > gpurun_out/ncu_bwd.log 2>&1
tail -2 gpurun_out/ncu_fwd.log gpurun_out/ncu_bwd.log
