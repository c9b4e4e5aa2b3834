# Builds the in-tree C-ABI library paper_1711_07240_b200/libcgbn.so for sm_100a.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -std=c++17 $(ARCH) -lineinfo -Xcompiler -fPIC -Iinclude --expt-relaxed-constexpr
PKG := paper_1711_07240_b200
LIB := $(PKG)/libcgbn.so
SRCS := $(PKG)/csrc/cgbn.cu
HDRS := $(wildcard $(PKG)/csrc/*.cuh) include/cgbn.h

all: $(LIB)

$(LIB): $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) -Xptxas -v -shared -o $@ $(SRCS) 2> $(PKG)/csrc/ptxas.log || (cat $(PKG)/csrc/ptxas.log; exit 1)

sass: $(LIB)
	cuobjdump -sass $(LIB) > $(PKG)/csrc/cgbn.sass

clean:
	rm -f $(LIB)

.PHONY: all clean sass
