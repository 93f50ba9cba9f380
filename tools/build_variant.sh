#!/bin/bash
# Build libisax.so with extra nvcc flags into variants/<name>/libisax.so (A/B measurement; run
# with ISAX_LIB=variants/<name>/libisax.so). Usage: bash tools/build_variant.sh <name> "<flags>"
set -e
cd "$(dirname "$0")/.."
name=$1; flags=$2
od=variants/$name; mkdir -p $od/obj
ARCH="-gencode arch=compute_100a,code=sm_100a"
pids=()
for s in paper_2009_01614_b200/csrc/*.cu; do
  /usr/local/cuda/bin/nvcc $ARCH -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -Xptxas -v,-warn-spills -I include $flags \
    -c $s -o $od/obj/$(basename $s .cu).o > $od/obj/$(basename $s .cu).log 2>&1 &
  pids+=($!)
done
for p in ${pids[@]}; do wait $p || { cat $od/obj/*.log | grep -i error | head; exit 1; }; done
/usr/local/cuda/bin/nvcc $ARCH -shared -Xcompiler -fPIC $od/obj/*.o -ldl -o $od/libisax.so
grep -h "spill stores" $od/obj/*.log | grep -v " 0 bytes spill" | head -3
echo "$od/libisax.so"
