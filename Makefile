# Build of the B200-native library (sm_100a) and the test-infrastructure
# oracles. `make -j` builds everything; __graft_entry__.build() calls it.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
EXTRA ?=
NVFLAGS := $(ARCH) -O3 -lineinfo $(EXTRA) -std=c++17 -Xcompiler -fPIC -Iinclude -Ipaper_2505_06771_b200/csrc \
           -Xptxas -warn-spills --expt-relaxed-constexpr
PKG := paper_2505_06771_b200
SRC := $(wildcard $(PKG)/csrc/*.cu)
OBJDIR ?= build/obj
OBJ := $(patsubst $(PKG)/csrc/%.cu,$(OBJDIR)/%.o,$(SRC))
HDR := $(wildcard $(PKG)/csrc/*.cuh $(PKG)/csrc/*.h) include/mrsim_cuda.h
LIB ?= $(PKG)/libmrsim_cuda.so

all: $(LIB) oracle

$(LIB): $(OBJ)
	@mkdir -p $(dir $@)
	$(NVCC) $(ARCH) -shared -cudart static -o $@ $(OBJ)

$(OBJDIR)/%.o: $(PKG)/csrc/%.cu $(HDR)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c $< -o $@

oracle: $(LIB)
	$(MAKE) -C oracle all

clean:
	rm -rf build $(LIB)

.PHONY: all oracle clean
