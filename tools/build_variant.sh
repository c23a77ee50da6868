#!/bin/bash
# Build a libgcm variant with extra defines, e.g.: tools/build_variant.sh trace4 -DGCM_TRACE -DGCM_LOOKC=4
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
name=$1; shift
NCCL=$(python -c "import nvidia.nccl,os;print(list(nvidia.nccl.__path__)[0])")
mkdir -p "$ROOT/paper_1011_1173_b200/lib/variants"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared "$@" \
  -I "$ROOT/include" -I "$NCCL/include" -DGCM_WITH_NCCL=1 "$ROOT"/paper_1011_1173_b200/csrc/*.cu \
  -L "$NCCL/lib" -l:libnccl.so.2 -Xlinker -rpath="$NCCL/lib" -o "$ROOT/paper_1011_1173_b200/lib/variants/libgcm_$name.so"
echo "$ROOT/paper_1011_1173_b200/lib/variants/libgcm_$name.so"
