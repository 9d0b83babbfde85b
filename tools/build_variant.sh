#!/usr/bin/env bash
# Build paper_2508_10395_b200/libxquant_<name>.so with extra nvcc flags, for A/B
# experiments on the GPU box (select with XQ_LIB=<path>).
#   bash tools/build_variant.sh kh2s3 -DXQ_KH2_STAGES=3 -DXQ_CSTAGES_MAX=8
set -eu
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; shift
OBJ=$ROOT/build/obj_$NAME
mkdir -p "$OBJ"
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -I $ROOT/include $*"
pids=()
for f in "$ROOT"/paper_2508_10395_b200/csrc/*.cu; do
  $NVCC $FL -c "$f" -o "$OBJ/$(basename "$f").o" & pids+=($!)
done
for p in "${pids[@]}"; do wait "$p"; done
$NVCC -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o "$ROOT/paper_2508_10395_b200/libxquant_$NAME.so" "$OBJ"/*.o
echo built "$ROOT/paper_2508_10395_b200/libxquant_$NAME.so"
