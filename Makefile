# Build the B200-native library (sm_100a) and the parity checkers.
#   make            -> paper_2110_14934_b200/librgbdseg_b200.so + oracle
#   make lib        -> the CUDA library only
NVCC     ?= nvcc
ARCH     := -gencode arch=compute_100a,code=sm_100a
# IEEE binary32 exactly as the reference CPU build: no FMA contraction, IEEE
# div/sqrt, denormals kept.  No --use_fast_math.
NVFLAGS  := $(ARCH) -O3 -lineinfo -std=c++17 -fmad=false -prec-div=true -prec-sqrt=true \
            -ftz=false -Xcompiler -fPIC,-O2 -Xptxas -warn-spills
PKG      := paper_2110_14934_b200
CSRC     := $(PKG)/csrc
LIB      := $(PKG)/librgbdseg_b200.so
OBJS     := $(CSRC)/rgbdseg_kernels.o $(CSRC)/rgbdseg_capi.o

all: lib oracle

lib: $(LIB)

$(CSRC)/%.o: $(CSRC)/%.cu $(CSRC)/gmm_pixel.cuh $(CSRC)/rgbdseg_kernels.cuh $(CSRC)/k1_experiments.cuh include/rgbdseg_c.h
	$(NVCC) $(NVFLAGS) -c $< -o $@

# cudart is linked shared (libcudart.so.12, the process's one CUDA runtime).
$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -cudart shared -o $@ $(OBJS)

oracle:
	$(MAKE) -C oracle $(if $(wildcard /root/reference/proj/src),all,$(CURDIR)/oracle/liboracle.so)

clean:
	rm -f $(CSRC)/*.o $(LIB)
	$(MAKE) -C oracle clean

.PHONY: all lib oracle clean
