#!/usr/bin/env bash
# Build paper_2508_10395_b200/libxquant_prof${XQ_SUFFIX:-}.so with -DXQ_ROLE_PROFILE (per-role
# barrier wait counters in the absorbed kernel). Use it with XQ_LIB=<path>.
set -eu
ROOT=$(cd "$(dirname "$0")/.." && pwd)
OBJ=$ROOT/build/obj_prof${XQ_SUFFIX:-}
mkdir -p "$OBJ"
NVCC=${NVCC:-/usr/local/cuda/bin/nvcc}
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -DXQ_ROLE_PROFILE -I $ROOT/include ${XQ_EXTRA:-}"
pids=()
for f in "$ROOT"/paper_2508_10395_b200/csrc/*.cu; do
  $NVCC $FL -c "$f" -o "$OBJ/$(basename "$f").o" & pids+=($!)
done
for p in "${pids[@]}"; do wait "$p"; done
$NVCC -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o "$ROOT/paper_2508_10395_b200/libxquant_prof${XQ_SUFFIX:-}.so" "$OBJ"/*.o
echo built "$ROOT/paper_2508_10395_b200/libxquant_prof${XQ_SUFFIX:-}.so"
