# Top-level build: every native artefact of the repo (run by __graft_entry__.build()).
#   paper_1905_04341_b200/lib/libpmhd_host.so        host C++ layer (pmhd_host.h)
#   paper_1905_04341_b200/lib/libpmhd_gpu.so         CUDA C-ABI, sm_100a, FMA build (product)
#   paper_1905_04341_b200/lib/libpmhd_gpu_parity.so  same sources, --fmad=false (bitwise parity runs)
#   paper_1905_04341_b200/bin/pmhd                   C++ CLI (run / bench) over the two libraries
#   oracle/liboracle.so (+ oracle/_ref/)             CPU oracle -- test infrastructure
NVCC     ?= nvcc
HOSTCXX  ?= g++
PKG      := paper_1905_04341_b200
LIB      := $(PKG)/lib
GPUSRC   := $(PKG)/csrc/gpu
ARCH     := -gencode arch=compute_100a,code=sm_100a
NVFLAGS  := $(ARCH) -O3 -lineinfo -Xlinker -Bsymbolic -std=c++17 -Xcompiler -fPIC -Xcompiler -O3 -Iinclude -I$(GPUSRC) \
            -Xptxas -warn-spills --expt-relaxed-constexpr
HOSTFLAGS:= -std=c++20 -O2 -march=x86-64-v3 -fPIC -Wall -Wextra -Iinclude
GPU_SRCS := $(GPUSRC)/pmhd_gpu.cu $(GPUSRC)/kernels_split.cu $(GPUSRC)/kernels_flux.cu $(GPUSRC)/kernels_update.cu $(GPUSRC)/kernels_update_tma.cu $(GPUSRC)/kernels_update_ws.cu $(GPUSRC)/kernels_update_emf.cu $(GPUSRC)/kernels_halo.cu $(GPUSRC)/kernels_drive.cu $(GPUSRC)/kernels_ctl.cu
# product division / sqrt: MUFU seed + one cubic Newton step, within 1 ulp
# (tests/test_divsqrt.py); -DPMHD_FAST_DIVSQRT alone is the IEEE-exact variant
FASTDS   := -DPMHD_FAST_DIVSQRT -DPMHD_DIVSQRT_1ULP
GPU_DEPS := $(GPU_SRCS) $(wildcard $(GPUSRC)/*.cuh) include/pmhd_gpu.h Makefile

all: host gpu cli oracle testlib

host: $(LIB)/libpmhd_host.so
gpu: $(LIB)/libpmhd_gpu.so $(LIB)/libpmhd_gpu_parity.so

$(LIB)/libpmhd_host.so: $(PKG)/csrc/host/pmhd_host.cpp $(PKG)/csrc/host/snapshot.cpp $(PKG)/csrc/host/perf_model.cpp include/pmhd_host.h include/pmhd_gpu.h
	@mkdir -p $(LIB)
	$(HOSTCXX) $(HOSTFLAGS) -shared -o $@ $(PKG)/csrc/host/pmhd_host.cpp $(PKG)/csrc/host/snapshot.cpp $(PKG)/csrc/host/perf_model.cpp

$(LIB)/libpmhd_gpu.so: $(GPU_DEPS)
	@mkdir -p $(LIB)
	$(NVCC) $(NVFLAGS) $(FASTDS) -shared -o $@ $(GPU_SRCS)

$(LIB)/libpmhd_gpu_parity.so: $(GPU_DEPS)
	@mkdir -p $(LIB)
	$(NVCC) $(NVFLAGS) --fmad=false -DPMHD_PARITY -shared -o $@ $(GPU_SRCS)

# GPU test helper (tests/cuda): checks the product build's division / sqrt
testlib: $(LIB)/test/libpmhd_divsqrt_check.so $(LIB)/test/libpmhd_divsqrt_exact_check.so \
         $(LIB)/test/libpmhd_gpu_check.so

$(LIB)/test/libpmhd_divsqrt_exact_check.so: tests/cuda/divsqrt_check.cu $(GPUSRC)/physics.cuh Makefile
	@mkdir -p $(LIB)/test
	$(NVCC) $(NVFLAGS) -DPMHD_FAST_DIVSQRT -shared -o $@ $<

# bounds-checked debug build of the product (tests/test_gpu_bounds.py)
$(LIB)/test/libpmhd_gpu_check.so: $(GPU_DEPS)
	@mkdir -p $(LIB)/test
	$(NVCC) $(NVFLAGS) $(FASTDS) -DPMHD_BOUNDS_CHECK -shared -o $@ $(GPU_SRCS)

$(LIB)/test/libpmhd_divsqrt_check.so: tests/cuda/divsqrt_check.cu $(GPUSRC)/physics.cuh Makefile
	@mkdir -p $(LIB)/test
	$(NVCC) $(NVFLAGS) $(FASTDS) -shared -o $@ $<

cli: $(PKG)/bin/pmhd

$(PKG)/bin/pmhd: $(PKG)/csrc/host/pmhd_cli.cpp $(LIB)/libpmhd_host.so $(LIB)/libpmhd_gpu.so
	@mkdir -p $(PKG)/bin
	$(HOSTCXX) $(HOSTFLAGS) -o $@ $< -L$(LIB) -lpmhd_host -l:libpmhd_gpu.so -Wl,-rpath,'$$ORIGIN/../lib'

oracle:
	$(MAKE) -C oracle CXX=$(HOSTCXX)

clean:
	rm -f $(LIB)/*.so
	$(MAKE) -C oracle clean

.PHONY: all host gpu cli oracle clean exp testlib

# A/B experiment builds (bench.py honours PMHD_GPU_LIB=<path>)
exp: $(GPU_DEPS)
	@mkdir -p $(LIB)/exp
	$(NVCC) $(NVFLAGS) $(FASTDS) -DPMHD_FLUX_SMEMW=0 -DPMHD_FLUX_MINB=4 -shared -o $(LIB)/exp/libpmhd_gpu_regs.so $(GPU_SRCS)
	$(NVCC) $(NVFLAGS) $(FASTDS) -DPMHD_FLUX_MINB=4 -shared -o $(LIB)/exp/libpmhd_gpu_minb4.so $(GPU_SRCS)
	$(NVCC) $(NVFLAGS) $(FASTDS) -DPMHD_FLUX_MINB=6 -shared -o $(LIB)/exp/libpmhd_gpu_minb6.so $(GPU_SRCS)
