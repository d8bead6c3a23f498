# Builds libmdc.so (sm_100a) in-tree and the CPU parity oracle.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
           -diag-suppress 550
PKG := paper_1408_0677_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
OBJ := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRC))

all: $(PKG)/libmdc.so oracle

build/%.o: $(PKG)/csrc/%.cu $(wildcard $(PKG)/csrc/*.cuh) include/mdc.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -c $< -o $@

# the seam kernels mirror numba's operation order: no FMA contraction
build/seam.o: NVFLAGS += -fmad=false
build/linear.o: NVFLAGS += -fmad=false

$(PKG)/libmdc.so: $(OBJ)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJ)

oracle:
	$(MAKE) -s -C oracle

clean:
	rm -rf build $(PKG)/libmdc.so

.PHONY: all oracle clean
