# Build the B200 C-ABI library (in-tree, travels to the GPU box) and the CPU oracle.
NVCC ?= /usr/local/cuda/bin/nvcc
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v
PKG := paper_2402_10517_b200
SRCS := $(PKG)/csrc/apb_abi.cu $(PKG)/csrc/apb_bitplane.cu $(PKG)/csrc/apb_gemv.cu $(PKG)/csrc/apb_gemv7.cu $(PKG)/csrc/apb_decode.cu $(PKG)/csrc/apb_quant.cu $(PKG)/csrc/apb_peer.cu $(PKG)/csrc/apb_dense.cu $(PKG)/csrc/apb_dense_tc.cu
OBJS := $(SRCS:.cu=.o)
LIB := $(PKG)/libanyprec_b200.so

all: $(LIB) oracle/liboracle.so

$(PKG)/csrc/%.o: $(PKG)/csrc/%.cu $(PKG)/csrc/apb_common.cuh include/anyprec_b200.h
	$(NVCC) $(NVFLAGS) -c $< -o $@ 2> $@.ptxas.log || (cat $@.ptxas.log; false)

# the quantizer is bit-exact with the reference's float64 numpy arithmetic: no FMA contraction
$(PKG)/csrc/apb_quant.o: NVFLAGS += -fmad=false

$(LIB): $(OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -lcudart

oracle/liboracle.so: oracle/anyprec_oracle.c
	gcc -O2 -march=x86-64-v2 -fPIC -shared -pthread -o $@ $<

clean:
	rm -f $(OBJS) $(LIB) oracle/liboracle.so $(PKG)/csrc/*.ptxas.log

.PHONY: all clean
