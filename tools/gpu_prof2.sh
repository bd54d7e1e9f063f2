set -x
python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
for o in "" "--opt halo=48" "--opt halo=40" "--opt tile=16" "--opt tile=64 --opt halo=96" "--opt cpt=4" "--opt cpt=4 --opt halo=40"; do
  python tools/prof.py --config 4 --sweeps 3 --time $o 2>&1 | tail -2
done
for o in "" "--opt halo=80" "--opt tile=16" "--opt cpt=4"; do
  python tools/prof.py --config 5 --sweeps 3 --time $o 2>&1 | tail -2
done
python tools/prof.py --config 3 --sweeps 3 --time 2>&1 | tail -2
