# Builds libpipefill.so (sm_100a only) and the oracle's C helpers.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -Xptxas -v --expt-relaxed-constexpr
PKG := paper_2410_07192_b200
SRCS := $(wildcard $(PKG)/csrc/*.cu)
HDRS := $(wildcard $(PKG)/csrc/*.cuh) $(wildcard $(PKG)/csrc/*.h) include/pipefill.h
LIB := $(PKG)/libpipefill.so

all: $(LIB)

$(LIB): $(SRCS) $(HDRS)
	$(NVCC) $(NVFLAGS) -shared -o $@ $(SRCS) 2> build/ptxas.log || (cat build/ptxas.log; exit 1)

$(shell mkdir -p build)

clean:
	rm -f $(LIB)

.PHONY: all clean
