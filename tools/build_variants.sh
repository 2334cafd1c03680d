#!/bin/bash
# Build tuning variants of the library into build_variants/<name>/ (experiments only).
set -e
cd "$(dirname "$0")/.."
declare -A V
V[ha]=""
V[hb]="-DHECNN_GM_TAPB=2"
V[hc]="-DHECNN_GM_TAPB=2 -DHECNN_GM_MINB=1"
V[hd]="-DHECNN_GM_OCT=4 -DHECNN_GM_MINB=3"
V[he]="-DHECNN_GM_TAPB=2 -DHECNN_GM_TPB=128 -DHECNN_GM_MINB=4"
V[hf]="-DHECNN_GM_OCT=4 -DHECNN_GM_TAPB=8 -DHECNN_GM_MINB=3"
for name in "${!V[@]}"; do
  [ -n "$1" ] && [[ ! " $* " =~ " $name " ]] && continue
  make -s -C paper_1911_11377_b200/csrc -j8 OUT=$PWD/build_variants/$name OBJ=$PWD/build_variants/$name/obj EXTRA_NVFLAGS="${V[$name]}" >/dev/null
  echo "built $name: ${V[$name]}"
done
