# Builds the product library (sm_100a) and the oracle (test infrastructure).
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -O3
PKG := paper_2205_05982_b200
BUILD := build
HDRS := $(wildcard $(PKG)/csrc/*.cuh) include/vxsort_b200.h

all: $(PKG)/lib/libvxsort_b200.so checked oracle

# sort kernels + single-GPU host orchestration (the long compile)
$(BUILD)/vxsort_b200.o: $(PKG)/csrc/vxsort_b200.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c -o $@ $<

# distributed sample sort (host orchestration over the C ABI; NCCL via dlopen)
$(BUILD)/dist_sort.o: $(PKG)/csrc/dist_sort.cu include/vxsort_b200.h
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -c -o $@ $<

$(PKG)/lib/libvxsort_b200.so: $(BUILD)/vxsort_b200.o $(BUILD)/dist_sort.o
	@mkdir -p $(PKG)/lib
	$(NVCC) $(ARCH) -shared -o $@ $^ -ldl

# checked build: device-side bounds / consistency checks (VXS_CHECKS); the
# tests run a parity subset against it (VXSORT_LIB=checked)
checked: $(PKG)/lib/libvxsort_b200_checked.so

$(BUILD)/vxsort_b200_checked.o: $(PKG)/csrc/vxsort_b200.cu $(HDRS)
	@mkdir -p $(BUILD)
	$(NVCC) $(NVFLAGS) -DVXS_CHECKS -c -o $@ $<

$(PKG)/lib/libvxsort_b200_checked.so: $(BUILD)/vxsort_b200_checked.o $(BUILD)/dist_sort.o
	@mkdir -p $(PKG)/lib
	$(NVCC) $(ARCH) -shared -o $@ $^ -ldl

oracle:
	$(MAKE) -C oracle

clean:
	rm -rf $(PKG)/lib/*.so $(BUILD)
	$(MAKE) -C oracle clean

.PHONY: all checked oracle clean
