#!/bin/bash
# Developer A/B: build libdjg.so with extra -D flags into
# paper_2106_14189_b200/_build_<name>/ (git-ignored, travels to the GPU box);
# select it with DJG_LIB_PATH=paper_2106_14189_b200/_build_<name>/libdjg.so.
#   tools/build_variant.sh <name> -DDJG_WIN_FILL=1 ...
set -e
name=$1; shift
R=$(cd "$(dirname "$0")/.." && pwd)
C=$R/paper_2106_14189_b200/csrc
O=$R/paper_2106_14189_b200/_build_$name
mkdir -p "$O"
make -s -C "$C" "$R/paper_2106_14189_b200/_build/scenario.o"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 \
  -Xcompiler -fPIC,-fopenmp,-ffp-contract=off -I"$R/include" -I"$C/cuda" "$@" -c "$C/cuda/engine.cu" -o "$O/engine.o"
METIS=$(ls /usr/local/cuda/targets/x86_64-linux/lib/libmetis_static.a 2>/dev/null || true)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fopenmp -o "$O/libdjg.so" "$O/engine.o" \
  "$R/paper_2106_14189_b200/_build/scenario.o" $METIS -lgomp
echo "built $O/libdjg.so"
