# libfdp.so: sm_100a kernels + host numerics + C ABI (include/fdp.h).
NVCC ?= /usr/local/cuda/bin/nvcc
PKG := paper_1712_00403_b200
SRC := $(PKG)/csrc
LIB := $(PKG)/libfdp.so
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 --expt-relaxed-constexpr
OBJ := build/mode_tma.o build/abi_tma.o build/mode_contract.o build/mode_small.o build/mode_plane.o build/kron_band.o build/kron_mass.o build/slab.o build/vec.o build/abi.o build/abi_block.o build/abi_slab.o build/abi_iga.o build/abi_kron.o build/abi_krylov.o build/host_eig.o build/host_iga.o build/host_geo.o build/nccl_dl.o
HDR := $(SRC)/fdp_internal.h $(SRC)/abi_impl.h $(SRC)/mode_tma.h include/fdp.h

all: $(LIB)

build/%.o: $(SRC)/kernels/%.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -Xptxas -v -c $< -o $@ 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

build/%.o: $(SRC)/%.cpp $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -x cu -c $< -o $@

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJ) -ldl

# diagnostic library (K1t per-role clock64 totals, fdp_k1t_prof_read); load with
# FDP_LIB_PATH=paper_1712_00403_b200/libfdp_prof.so
PROFLIB := $(PKG)/libfdp_prof.so
prof: $(PROFLIB)
build/prof_mode_tma.o: $(SRC)/kernels/mode_tma.cu $(HDR)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -DFDP_K1T_PROF -c $< -o $@
$(PROFLIB): build/prof_mode_tma.o $(filter-out build/mode_tma.o,$(OBJ))
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $^ -ldl

clean:
	rm -rf build $(LIB) $(PROFLIB)

.PHONY: all clean prof
