#!/bin/bash
# Builds libvpb variants for tuning sweeps:
# NAME = <min CTAs/SM>_<window cap>[_<staged candidates>[_<smem carveout %, -1 auto>[_<line prefilter 0|1>]]].
set -e
cd "$(dirname "$0")/.."
mkdir -p build/variants
for v in "$@"; do
  IFS=_ read -r b c cc co pf <<< "$v"
  cc=${cc:-160}
  co=${co:--1}
  pf=${pf:-0}
  [ "$pf" = 1 ] && pfv=true || pfv=false
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC,-ffp-contract=off \
    -DVPB_MARCH_MINB=$b -DVPB_WINDOW_CAP=$c -DVPB_CAND_CAP=$cc -DVPB_CARVEOUT=$co -DVPB_NORMAL_PF=$pfv -c paper_2103_01954_b200/csrc/vpb_kernels.cu \
    -o build/variants/k_$v.o -Xptxas -v 2> build/variants/k_$v.log
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/variants/libvpb_$v.so build/variants/k_$v.o \
    build/obj/vpb_backward.o build/obj/vpb_train.o build/obj/vpb_compose.o build/obj/vpb_bvh.o build/obj/vpb_api.o build/obj/vpb_synth.o build/obj/vpb_losses.o -cudart static
  echo "$v: $(grep -A2 'k_march_tilesILi' build/variants/k_$v.log | grep -oE 'Used [0-9]+ registers|[0-9]+ bytes spill stores' | head -2 | tr '\n' ' ')"
done
