# Top-level build: the product library (sm_100a only) and the CPU checkers.
#
#   make            -> paper_2405_15593_b200/lib/libmicroadam_cuda.so  + oracle/
#   make lib        -> the CUDA library only
#   make oracle     -> oracle/_build/liboracle.so (+ oracle/_ref when /root/reference exists)
NVCC     ?= /usr/local/cuda/bin/nvcc
PKG      := paper_2405_15593_b200
CSRC     := $(PKG)/csrc
LIBDIR   ?= $(PKG)/lib
LIB      := $(LIBDIR)/libmicroadam_cuda.so
# -fmad=false: no FMA contraction anywhere on device (bit-exact fp64 EF path).
NVFLAGS  := -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo \
            -fmad=false -Xcompiler -fPIC -Xcompiler -ffp-contract=off \
            -Xcompiler -fvisibility=hidden -Xptxas -warn-spills $(EXTRA)
SRCS     := $(CSRC)/ma_nccl.cpp $(CSRC)/ma_bigblock.cu $(CSRC)/ma_kernels.cu $(CSRC)/ma_fast.cu $(CSRC)/ma_warp.cu $(CSRC)/ma_tile.cu $(CSRC)/ma_global.cu $(CSRC)/ma_capi.cu $(CSRC)/microadam_b200.cpp
HDRS     := include/microadam_cuda.h include/ma_synth.h $(CSRC)/ma_internal.h $(CSRC)/ma_device.cuh $(CSRC)/ma_async.cuh $(CSRC)/microadam_b200.hpp

.PHONY: all lib oracle clean sass
all: lib oracle

lib: $(LIB)

$(LIBDIR)/%.o: $(CSRC)/%.cu $(HDRS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(NVFLAGS) -Iinclude -dc -o $@ $<

$(LIBDIR)/%.o: $(CSRC)/%.cpp $(HDRS)
	@mkdir -p $(LIBDIR)
	$(NVCC) $(NVFLAGS) -Iinclude -x cu -dc -o $@ $<

$(LIB): $(LIBDIR)/ma_nccl.o $(LIBDIR)/ma_bigblock.o $(LIBDIR)/ma_kernels.o $(LIBDIR)/ma_fast.o $(LIBDIR)/ma_warp.o $(LIBDIR)/ma_tile.o $(LIBDIR)/ma_global.o $(LIBDIR)/ma_capi.o $(LIBDIR)/microadam_b200.o
	$(NVCC) $(NVFLAGS) -shared -o $@ $^ -ldl

oracle: lib  # the adapter links the product library
	$(MAKE) -s -C oracle $(if $(wildcard /root/reference/proj/src),all,oracle)

sass: $(LIB)
	/usr/local/cuda/bin/cuobjdump -sass $(LIB) > $(LIBDIR)/libmicroadam_cuda.sass

clean:
	rm -rf $(LIBDIR)
	$(MAKE) -s -C oracle clean
