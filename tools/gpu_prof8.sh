for o in "" "--opt prefetch=1" "--opt order=0 --opt prefetch=1"; do
  python tools/prof.py --config 4 --sweeps 3 --time $o 2>&1 | tail -2
done
MMF_LIB=paper_2106_14485_b200/libmmf_b4.so python tools/prof.py --config 4 --sweeps 3 --time 2>&1 | tail -2
MMF_LIB=paper_2106_14485_b200/libmmf_b4.so python tools/prof.py --config 4 --sweeps 3 --time --opt prefetch=1 2>&1 | tail -2
for o in "" "--opt prefetch=1"; do python tools/prof.py --config 5 --sweeps 3 --time $o 2>&1 | tail -2; done
MMF_LIB=paper_2106_14485_b200/libmmf_b4.so python tools/prof.py --config 5 --sweeps 3 --time 2>&1 | tail -2
echo done
