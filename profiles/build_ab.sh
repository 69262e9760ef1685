#!/bin/bash
# Build A/B variants of merge.cu (compile-time knobs) as whole libraries under build_ab/:
#   profiles/build_ab.sh NAME "-DKNOB=V ..."  ->  build_ab/libvdi_NAME.so  (select with VDI_LIB_PATH)
#   SRC=path/to/merge.cu profiles/build_ab.sh NAME ""  builds another revision of merge.cu (includes resolve from csrc/)
set -e
NAME=$1; DEFS=$2
SP=$(python -c "import site; print(site.getsitepackages()[0])")
NCCL=$SP/nvidia/nccl
ARCH="-gencode arch=compute_100a,code=sm_100a"
mkdir -p build_ab
make -s all >/dev/null
nvcc -std=c++17 -O3 $ARCH -lineinfo -fmad=false -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -Iinclude \
  -I$NCCL/include $DEFS -dc -o build_ab/merge_$NAME.o ${SRC:-paper_2206_14503_b200/csrc/merge.cu}
nvcc $ARCH -shared -o build_ab/libvdi_$NAME.so build/api.o build_ab/merge_$NAME.o build/generate.o build/comm.o \
  build/render.o -L$NCCL/lib -l:libnccl.so.2 -Xlinker -rpath -Xlinker $NCCL/lib
echo build_ab/libvdi_$NAME.so
