# Builds libpipefill.so (sm_100a only): one object per translation unit (parallel with -j),
# then one shared link.
NVCC ?= nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 -Xptxas -v --expt-relaxed-constexpr
PKG := paper_2410_07192_b200
SRCS := $(wildcard $(PKG)/csrc/*.cu)
OBJS := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRCS))
HDRS := $(wildcard $(PKG)/csrc/*.cuh) $(wildcard $(PKG)/csrc/*.h) include/pipefill.h
LIB := $(PKG)/libpipefill.so

all: $(LIB)

build/%.o: $(PKG)/csrc/%.cu $(HDRS) | build
	$(NVCC) $(NVFLAGS) -c -o $@ $< 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; exit 1)

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS)

build:
	mkdir -p build

clean:
	rm -f $(LIB) $(OBJS)

.PHONY: all clean
