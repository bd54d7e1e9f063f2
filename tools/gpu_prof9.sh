for lib in libmmf libmmf_b3u84 libmmf_b2u84 libmmf_b3u44; do
  echo "== $lib"
  MMF_LIB=paper_2106_14485_b200/$lib.so python tools/prof.py --config 4 --sweeps 3 --time --opt order=0 2>&1 | tail -1
  MMF_LIB=paper_2106_14485_b200/$lib.so python tools/prof.py --config 4 --sweeps 3 --time --opt order=0 --opt cpt=4 2>&1 | tail -1
  MMF_LIB=paper_2106_14485_b200/$lib.so python tools/prof.py --config 5 --sweeps 3 --time 2>&1 | tail -1
done
echo done
