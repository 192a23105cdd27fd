# Build of the B200-native library (sm_100a) and the test-infrastructure
# oracles. `make -j` builds everything; __graft_entry__.build() calls it.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Iinclude -Ipaper_2505_06771_b200/csrc \
           -Xptxas -warn-spills --expt-relaxed-constexpr
PKG := paper_2505_06771_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
OBJ := $(patsubst $(PKG)/csrc/%.cu,build/obj/%.o,$(SRC))
HDR := $(wildcard $(PKG)/csrc/*.cuh $(PKG)/csrc/*.h) include/mrsim_cuda.h
LIB := $(PKG)/libmrsim_cuda.so

all: $(LIB) oracle

$(LIB): $(OBJ)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJ)

build/obj/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p build/obj
	$(NVCC) $(NVFLAGS) -c $< -o $@

oracle: $(LIB)
	$(MAKE) -C oracle all

clean:
	rm -rf build $(LIB)

.PHONY: all oracle clean
