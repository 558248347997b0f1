# usage: build_variant2.sh NAME "extra nvcc flags" — rebuilds vpb_kernels.cu and vpb_backward.cu
# with the flags (tuning sweeps of the ray-batch kernels); output build/variants/libvpb_NAME.so
cd /root/repo
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -prec-div=true -prec-sqrt=true -Xcompiler -fPIC,-ffp-contract=off -Xptxas -v"
mkdir -p build/variants
nvcc $F $2 -c paper_2103_01954_b200/csrc/vpb_kernels.cu -o build/variants/k_$1.o 2> build/variants/k_$1.log &
nvcc $F $2 -c paper_2103_01954_b200/csrc/vpb_backward.cu -o build/variants/b_$1.o 2> build/variants/b_$1.log &
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build/variants/libvpb_$1.so build/variants/k_$1.o build/variants/b_$1.o build/obj/vpb_train.o build/obj/vpb_compose.o build/obj/vpb_bvh.o build/obj/vpb_api.o build/obj/vpb_synth.o build/obj/vpb_losses.o -cudart static
echo "$1: $(grep -A2 'k_backward_rays_warp' build/variants/b_$1.log | grep -oE 'Used [0-9]+ registers|[0-9]+ bytes spill stores' | head -2 | tr '\n' ' ')"
