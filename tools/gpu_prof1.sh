set -x
python tools/prof.py --config 4 --sweeps 3 --time > gpurun_out/p_bis32.log 2>&1
python tools/prof.py --config 4 --sweeps 3 --time --opt tile=16 > gpurun_out/p_bis16.log 2>&1
python tools/prof.py --config 4 --sweeps 3 --time --opt tile=64 > gpurun_out/p_bis64.log 2>&1
python tools/prof.py --config 4 --sweeps 3 --time --opt cpt=4 > gpurun_out/p_cpt4.log 2>&1
python tools/prof.py --config 4 --sweeps 3 --time --opt cpt=1 > gpurun_out/p_cpt1.log 2>&1
python tools/prof.py --config 5 --sweeps 3 --time > gpurun_out/p_c5.log 2>&1
cat gpurun_out/p_*.log
python tools/prof.py --config 4 --sweeps 1 > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_fwd_tile -s 30 -c 1 -o gpurun_out/prof_fwd python tools/prof.py --config 4 --sweeps 1 > gpurun_out/ncu_fwd.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_bwd_tile -s 30 -c 1 -o gpurun_out/prof_bwd python tools/prof.py --config 4 --sweeps 1 > gpurun_out/ncu_bwd.log 2>&1
tail -3 gpurun_out/ncu_fwd.log
