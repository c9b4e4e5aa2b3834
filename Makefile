# Builds the in-tree C-ABI library paper_1711_07240_b200/libcgbn.so for sm_100a.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Iinclude --expt-relaxed-constexpr
PKG := paper_1711_07240_b200
LIB := $(PKG)/libcgbn.so
HDRS := $(wildcard $(PKG)/csrc/*.cuh) include/cgbn.h
OBJS := build/cgbn.o build/cgbn_conv.o

all: $(LIB)

# two translation units: the BN kernels (cgbn.cu + its .cuh parts) and the tcgen05
# producer-fusion conv (cgbn_conv.cu)
build/cgbn.o: $(PKG)/csrc/cgbn.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -Xptxas -v -c -o $@ $< 2> $(PKG)/csrc/ptxas.log || (cat $(PKG)/csrc/ptxas.log; exit 1)

build/cgbn_conv.o: $(PKG)/csrc/cgbn_conv.cu include/cgbn.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -Xptxas -v -c -o $@ $< 2> $(PKG)/csrc/ptxas_conv.log || (cat $(PKG)/csrc/ptxas_conv.log; exit 1)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)

sass: $(LIB)
	cuobjdump -sass $(LIB) > $(PKG)/csrc/cgbn.sass

clean:
	rm -f $(LIB) $(OBJS)

.PHONY: all clean sass
