# Builds the product library (sm_100a) and the oracle (test infrastructure).
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC -Xcompiler -O3
PKG := paper_2205_05982_b200
SRCS := $(wildcard $(PKG)/csrc/*.cu) $(wildcard $(PKG)/csrc/*.cuh) include/vxsort_b200.h

all: $(PKG)/lib/libvxsort_b200.so oracle

$(PKG)/lib/libvxsort_b200.so: $(SRCS)
	@mkdir -p $(PKG)/lib
	$(NVCC) $(NVFLAGS) -o $@ $(PKG)/csrc/vxsort_b200.cu

oracle:
	$(MAKE) -C oracle

clean:
	rm -f $(PKG)/lib/*.so
	$(MAKE) -C oracle clean

.PHONY: all oracle clean
