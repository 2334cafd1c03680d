#!/bin/bash
# Build tuning variants of the library into build_variants/<name>/ (experiments only).
set -e
cd "$(dirname "$0")/.."
declare -A V
V[na]=""
V[u2]="-DHECNN_RESCALE_UNROLL=2"
V[u2m4]="-DHECNN_RESCALE_UNROLL=2 -DHECNN_RESCALE_MINB=4"
V[u4m4]="-DHECNN_RESCALE_UNROLL=4 -DHECNN_RESCALE_MINB=4"
V[m4]="-DHECNN_RESCALE_MINB=4"
for name in "${!V[@]}"; do
  [ -n "$1" ] && [[ ! " $* " =~ " $name " ]] && continue
  make -s -C paper_1911_11377_b200/csrc -j8 OUT=$PWD/build_variants/$name OBJ=$PWD/build_variants/$name/obj EXTRA_NVFLAGS="${V[$name]}" >/dev/null
  echo "built $name: ${V[$name]}"
done
