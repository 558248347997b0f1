# usage: bv.sh NAME "extra nvcc flags"
cd /root/repo
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -prec-div=true -prec-sqrt=true -Xcompiler -fPIC,-ffp-contract=off $2 -c paper_2103_01954_b200/csrc/vpb_kernels.cu -o build/variants/k_$1.o -Xptxas -v 2> build/variants/k_$1.log && \
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/variants/libvpb_$1.so build/variants/k_$1.o build/obj/vpb_backward.o build/obj/vpb_train.o build/obj/vpb_compose.o build/obj/vpb_bvh.o build/obj/vpb_api.o build/obj/vpb_synth.o build/obj/vpb_losses.o build/obj/vpb_comm.o -cudart static -ldl
echo "$1: $(grep -A2 'k_march_tilesILi16ELi16ELi0ELi64ELi3ELb0E' build/variants/k_$1.log | grep -oE 'Used [0-9]+ registers|[0-9]+ bytes spill stores' | head -2 | tr '\n' ' ')"
