#!/bin/bash
# Build tuning variants of the library into build_variants/<name>/ (experiments only).
set -e
cd "$(dirname "$0")/.."
declare -A V
V[na]=""
V[a3]="-DHECNN_RESCALE_MINB_ADD=3"
V[a2]="-DHECNN_RESCALE_MINB_ADD=2"
V[p6]="-DHECNN_RESCALE_MINB=6"
V[a5]="-DHECNN_RESCALE_MINB_ADD=5"
for name in "${!V[@]}"; do
  [ -n "$1" ] && [[ ! " $* " =~ " $name " ]] && continue
  make -s -C paper_1911_11377_b200/csrc -j8 OUT=$PWD/build_variants/$name OBJ=$PWD/build_variants/$name/obj EXTRA_NVFLAGS="${V[$name]}" >/dev/null
  echo "built $name: ${V[$name]}"
done
