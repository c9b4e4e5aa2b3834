# Builds the in-tree C-ABI library paper_1711_07240_b200/libcgbn.so for sm_100a.
#   make -j4      (the four translation units compile in parallel)
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Iinclude --expt-relaxed-constexpr
PKG := paper_1711_07240_b200
LIB := $(PKG)/libcgbn.so
HDRS := $(wildcard $(PKG)/csrc/*.cuh) include/cgbn.h
# the BN kernels: cgbn.cu (+ its .cuh parts) compiled once per activation dtype
# (cgbn.cu: fp32 + the dtype-independent entry points; cgbn_bf16.cu, cgbn_f16.cu), and the
# tcgen05 producer-fusion conv (cgbn_conv.cu)
OBJS := build/cgbn_a0.o build/cgbn_a1.o build/cgbn_a2.o build/cgbn_conv.o

all: $(LIB)

build/cgbn_a0.o: $(PKG)/csrc/cgbn.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -Xptxas -v -c -o $@ $< 2> $(PKG)/csrc/ptxas_a0.log || (cat $(PKG)/csrc/ptxas_a0.log; exit 1)

# separate source files, so each unit's anonymous namespace is its own
build/cgbn_a1.o: $(PKG)/csrc/cgbn_bf16.cu $(PKG)/csrc/cgbn.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -Xptxas -v -c -o $@ $< 2> $(PKG)/csrc/ptxas_a1.log || (cat $(PKG)/csrc/ptxas_a1.log; exit 1)

build/cgbn_a2.o: $(PKG)/csrc/cgbn_f16.cu $(PKG)/csrc/cgbn.cu $(HDRS)
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -Xptxas -v -c -o $@ $< 2> $(PKG)/csrc/ptxas_a2.log || (cat $(PKG)/csrc/ptxas_a2.log; exit 1)

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
