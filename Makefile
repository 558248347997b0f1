# Build of the product library (libvpb.so, sm_100a) and the test-only oracles.
NVCC     ?= /usr/local/cuda/bin/nvcc
ARCH     := -gencode arch=compute_100a,code=sm_100a
PKG      := paper_2103_01954_b200
SRC      := $(PKG)/csrc
OBJ      := build/obj
# -fmad=false + IEEE div/sqrt on the device, -ffp-contract=off on the host: the reference's
# binary32 operation sequence is reproduced exactly (see vpb_device.cuh).
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -fmad=false -prec-div=true -prec-sqrt=true \
            -Xcompiler -fPIC,-ffp-contract=off,-O3 -Xptxas -v
HDRS     := $(wildcard $(SRC)/*.h $(SRC)/*.hpp $(SRC)/*.cuh) include/vpb.h

.PHONY: all lib oracle clean examples
all: lib oracle
# a C++ multi-GPU caller of the C-ABI (integration/ring_multi_gpu.cpp)
examples: build/ring_multi_gpu
build/ring_multi_gpu: integration/ring_multi_gpu.cpp include/vpb.h $(PKG)/libvpb.so
	@mkdir -p build
	g++ -O2 -std=c++17 -Iinclude -I/usr/local/cuda/include $< -L$(PKG) -lvpb -L/usr/local/cuda/lib64 -lcudart \
	    -Wl,-rpath,'$$ORIGIN/../$(PKG)' -o $@
lib: $(PKG)/libvpb.so
oracle:
	$(MAKE) -C oracle all

$(OBJ)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $(OBJ)/$*.ptxas.log || (cat $(OBJ)/$*.ptxas.log; false)

$(OBJ)/%.o: $(SRC)/%.cpp $(HDRS)
	@mkdir -p $(OBJ)
	$(NVCC) $(NVFLAGS) -x c++ -c $< -o $@

# NCCL (multi-GPU C-ABI, vpb_comm.cpp) is not linked: vpb_comm.cpp binds libnccl.so.2 with
# dlopen at the first vp_comm_* call (torch's copy when torch is loaded), so rendering never
# loads NCCL and cannot shadow torch's newer one.
$(PKG)/libvpb.so: $(OBJ)/vpb_kernels.o $(OBJ)/vpb_backward.o $(OBJ)/vpb_train.o $(OBJ)/vpb_compose.o $(OBJ)/vpb_bvh.o $(OBJ)/vpb_api.o $(OBJ)/vpb_synth.o $(OBJ)/vpb_losses.o $(OBJ)/vpb_comm.o
	$(NVCC) $(ARCH) -shared -o $@ $^ -cudart static -ldl

clean:
	rm -rf build $(PKG)/libvpb.so
	$(MAKE) -C oracle clean
