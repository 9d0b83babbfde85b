#!/usr/bin/env bash
# On the GPU box: launch lists + ncu --set full of the dominant kernel for each config,
# summarised in place (tools/summarize_profiles.py with PROFILE_OUT under gpurun_out/);
# the .ncu-rep files are deleted afterwards (they exceed gpurun's 64 MiB return limit).
#   bash tools/gpu_profile_all.sh r02 c4 c3
set -u
TAG=$1; shift
export PROFILE_OUT=gpurun_out/profiles_$TAG
mkdir -p "$PROFILE_OUT" gpurun_out/prof
for c in "$@"; do
  bash tools/profile_round.sh gpurun_out/prof "$c"
  python tools/summarize_profiles.py gpurun_out/prof "$TAG" "$c" > "$PROFILE_OUT/summary_$c.log" 2>&1
  rm -f gpurun_out/prof/decode_full_"$c".ncu-rep
done
