#!/bin/bash
# A/B builds of liblbg with extra compile definitions: tools/build_variant.sh NAME "-DFOO -DBAR"
# -> paper_2303_11811_b200/build_NAME/liblbg.so (load it with LBG_LIB=...)
set -e
NAME=$1; EXTRA=$2
cd "$(dirname "$0")/../paper_2303_11811_b200"
PYSITE=$(python3 -c "import sysconfig; print(sysconfig.get_paths()['purelib'])")
NCCL=$PYSITE/nvidia/nccl
OUT=build_$NAME
mkdir -p $OUT
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC,-ffp-contract=off,-O2 -I../include -I$NCCL/include $EXTRA"
pids=()
for f in csrc/*.cu; do
  b=$(basename $f .cu)
  /usr/local/cuda/bin/nvcc $FLAGS -c $f -o $OUT/$b.o & pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/liblbg.so $OUT/*.o -L$NCCL/lib -l:libnccl.so.2 -lcudart -Xlinker -rpath,$NCCL/lib
echo built $OUT/liblbg.so
