#!/bin/bash
# Build an experiment variant of the library: tools/build_variant.sh NAME "-DFLAG=..." [SRC_DIR]
# -> variants/NAME/libblest_b200.so (select at run time with BLEST_LIB=...; travels to the GPU box).
set -e
NAME=$1; FLAGS=$2; SRC=${3:-paper_2512_21967_b200/csrc}
OUT=variants/$NAME; OBJ=$(mktemp -d); mkdir -p $OUT
# (a source tree exported from another commit needs its ../../include next to it:
#  git archive <rev> paper_2512_21967_b200/csrc include | tar -x -C /tmp/x)
pids=()
for f in $SRC/*.cu; do
  b=$(basename $f .cu)
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
     --expt-relaxed-constexpr -Iinclude $FLAGS -c $f -o $OBJ/$b.o &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p || { echo "variant build failed" >&2; exit 1; }; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libblest_b200.so $OBJ/*.o -lcudart
rm -rf $OBJ
echo $OUT/libblest_b200.so
