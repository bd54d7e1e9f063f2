#!/bin/bash
# usage: tools/build_variant.sh NAME "-DFLAG=.. -DFLAG2=.."  -> paper_2106_14485_b200/libmmf_NAME.so
name=$1; shift
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -shared \
  --expt-relaxed-constexpr $@ -Xptxas -v -I include -o paper_2106_14485_b200/libmmf_$name.so \
  paper_2106_14485_b200/csrc/mmf.cu -ldl > /tmp/build_$name.log 2>&1 || { echo "build $name failed"; tail -5 /tmp/build_$name.log; exit 1; }
grep -A2 "k_fwd_wideINS_2TrIfsEELi8ELi1ELi0E\|k_bwd_wideINS_2TrIfsEELi8E" /tmp/build_$name.log | grep -E "Used|spill" | sed "s/^/$name: /"
