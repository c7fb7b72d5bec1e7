#!/bin/bash
# Build A/B variants of gc_o1.cu into abl/<name>.so (development tool; needs build/ from
# paper_1605_02178_b200.build).   usage: tools/abl_build.sh name1 "flags1" [src1] name2 "flags2" [src2] ...
#   src defaults to the working-tree gc_o1.cu; "HEAD" uses the committed one.
set -e
cd "$(dirname "$0")/.."
mkdir -p abl/obj
C=paper_1605_02178_b200/csrc
NCCL_LIB=$(python -c "import paper_1605_02178_b200.build as b; print(b._nccl_dirs()[1])")
NCCL_INC=$(python -c "import paper_1605_02178_b200.build as b; print(b._nccl_dirs()[0])")
OBJS=$(ls build/*.o | grep -v gc_o1.cu.o)
pids=()
while [ $# -gt 0 ]; do
  name=$1; flags=$2; src=${3:-$C/gc_o1.cu}; shift 3 || shift $#
  if [ "$src" = HEAD ]; then git show HEAD:$C/gc_o1.cu > abl/obj/${name}_src.cu; src=abl/obj/${name}_src.cu; fi
  ( /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
      -Iinclude -I$C -I$NCCL_INC $flags -c $src -o abl/obj/$name.o && \
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o abl/$name.so abl/obj/$name.o $OBJS \
      -L$NCCL_LIB -l:libnccl.so.2 -Xlinker -rpath,$NCCL_LIB -lcudart_static -lrt -ldl -lpthread && echo "built abl/$name.so" ) &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
