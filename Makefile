# Builds the product library (sm_100a CUDA + C-ABI) and the parity checkers.
#
#   make            -> paper_2512_13796_b200/libnexel_b200.so  (+ oracle/ checkers)
#   make lib        -> product only
#   make oracle     -> oracle/build/libnexel_oracle.so, oracle/_ref/*.so (if /root/reference exists)
#   make dropin     -> paper_2512_13796_b200/libnexel_dropin.so (C++ nexel::render shim;
#                      needs the reference's public headers)

NVCC ?= /usr/local/cuda/bin/nvcc
CXX ?= g++
ARCH := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -O3 -lineinfo -std=c++17 $(ARCH) -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr
REF ?= /root/reference/proj

PKG := paper_2512_13796_b200
SRC := $(PKG)/csrc
CU_SRCS := $(SRC)/nx_api.cu $(SRC)/nx_preprocess.cu $(SRC)/nx_sort.cu $(SRC)/nx_composite.cu $(SRC)/nx_texture.cu \
           $(SRC)/nx_texture_tc.cu
CPP_SRCS := $(SRC)/nx_synth.cpp
HDRS := include/nexel_b200.h $(SRC)/nx_internal.cuh $(SRC)/nx_sort.cuh
OBJDIR := build/obj
CU_OBJS := $(patsubst $(SRC)/%.cu,$(OBJDIR)/%.o,$(CU_SRCS))
CPP_OBJS := $(patsubst $(SRC)/%.cpp,$(OBJDIR)/%.o,$(CPP_SRCS))

.PHONY: all lib oracle dropin clean
all: lib oracle

lib: $(PKG)/libnexel_b200.so

$(OBJDIR)/%.o: $(SRC)/%.cu $(HDRS)
	@mkdir -p $(OBJDIR)
	$(NVCC) $(NVFLAGS) -c -o $@ $<

$(OBJDIR)/%.o: $(SRC)/%.cpp $(HDRS)
	@mkdir -p $(OBJDIR)
	$(CXX) -std=c++17 -O2 -fPIC -c -o $@ $<

$(PKG)/libnexel_b200.so: $(CU_OBJS) $(CPP_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $^ -Xlinker -Bsymbolic

oracle:
	$(MAKE) -C oracle REF=$(REF)

clean:
	rm -rf build $(PKG)/*.so
	$(MAKE) -C oracle clean
