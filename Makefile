# Builds libvdi.so (CUDA, sm_100a) and the CPU oracle's liboracle.so.
SP      := $(shell python -c "import site; print(site.getsitepackages()[0])")
NCCL    := $(SP)/nvidia/nccl
NVCC    ?= nvcc
ARCH    := -gencode arch=compute_100a,code=sm_100a
NVFLAGS := -std=c++17 -O3 $(ARCH) -lineinfo -fmad=false -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
           -Iinclude -I$(NCCL)/include -Xptxas -v
PKG     := paper_2206_14503_b200
SRCS    := $(PKG)/csrc/api.cu $(PKG)/csrc/merge.cu $(PKG)/csrc/generate.cu $(PKG)/csrc/comm.cu $(PKG)/csrc/render.cu
OBJS    := $(patsubst $(PKG)/csrc/%.cu,build/%.o,$(SRCS))
LIB     := $(PKG)/lib/libvdi.so

all: $(LIB) oracle/liboracle.so

build/%.o: $(PKG)/csrc/%.cu $(PKG)/csrc/internal.h $(PKG)/csrc/comm.h $(PKG)/csrc/render.h include/vdi.h
	@mkdir -p build
	$(NVCC) $(NVFLAGS) -dc -o $@ $< 2> build/$*.ptxas.log || (cat build/$*.ptxas.log; false)

$(LIB): $(OBJS)
	@mkdir -p $(PKG)/lib
	$(NVCC) $(ARCH) -shared -o $@ $(OBJS) -L$(NCCL)/lib -l:libnccl.so.2 -Xlinker -rpath -Xlinker $(NCCL)/lib

oracle/liboracle.so: oracle/oracle.cpp
	g++ -std=c++17 -O2 -ffp-contract=off -fno-fast-math -fopenmp -fPIC -shared -o $@ $<

# debug build with device-side bounds checks (VDI_CHECKS): build_dbg/libvdi.so;
# select it with VDI_LIB_PATH=$PWD/build_dbg/libvdi.so
DBG_OBJS := $(patsubst $(PKG)/csrc/%.cu,build_dbg/%.o,$(SRCS))
build_dbg/%.o: $(PKG)/csrc/%.cu $(PKG)/csrc/internal.h $(PKG)/csrc/comm.h $(PKG)/csrc/render.h include/vdi.h
	@mkdir -p build_dbg
	$(NVCC) $(NVFLAGS) -DVDI_CHECKS -dc -o $@ $< 2> build_dbg/$*.ptxas.log || (cat build_dbg/$*.ptxas.log; false)

build_dbg/libvdi.so: $(DBG_OBJS)
	$(NVCC) $(ARCH) -shared -o $@ $(DBG_OBJS) -L$(NCCL)/lib -l:libnccl.so.2 -Xlinker -rpath -Xlinker $(NCCL)/lib

debug: build_dbg/libvdi.so

clean:
	rm -rf build build_dbg $(LIB) oracle/liboracle.so

.PHONY: all clean debug
