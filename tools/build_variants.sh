#!/bin/bash
# Build tuning variants of the library into build_variants/<name>/ (experiments only).
set -e
cd "$(dirname "$0")/.."
declare -A V
V[na]=""
V[nb]="-DHECNN_KS_LOGB=12 -DHECNN_KS_MAXT_COL=256 -DHECNN_KS_MINB=2"
V[nc]="-DHECNN_KS_LOGB=12 -DHECNN_KS_MAXT_COL=512 -DHECNN_KS_MINB=2"
V[e4]="-DHECNN_KS_LOGE=4"
V[batch]="-DHECNN_NTT_BATCH=1"
V[nomac]="-DHECNN_KS_ABLATE_MAC"
V[nosplit]="-DHECNN_NTT_SPLIT=0"
V[col512]="-DHECNN_KS_MAXT_COL=512"
V[tcmin4]="-DHECNN_TC_MIN_KSTEPS=4"
V[rsu4]="-DHECNN_RESCALE_UNROLL=4"
V[pfcol]="-DHECNN_KS_PF_COL=1 -DHECNN_KS_MAXT_COL=512"
V[pfcol1k]="-DHECNN_KS_PF_COL=1"
V[n256m4]="-DHECNN_NTT_MAXT=256 -DHECNN_NTT_MINB=4"
V[n1024]="-DHECNN_NTT_MAXT=1024 -DHECNN_NTT_MINB=1"
V[ne4]="-DHECNN_NTT_LOGE=4"
V[notm]="-DHECNN_KS_TMEM=0"
V[tm2]="-DHECNN_KS_TMEM=2"
V[rsm6]="-DHECNN_RESCALE_MINB=6"
V[rsm8]="-DHECNN_RESCALE_MINB=8"
V[dm5]="-DHECNN_DIRECT_MINB=5"
V[dm6]="-DHECNN_DIRECT_MINB=6"
V[noepf]="-DHECNN_KS_EPI_PF=0"
V[kse4]="-DHECNN_KS_LOGE=4"
V[col512]="-DHECNN_KS_MAXT_COL=512"
V[g16]="-DHECNN_TC_G16=1"
V[kscl]="-DHECNN_KS_CLUSTER=1"
V[tc34]="-DHECNN_TC_STAGES=3 -DHECNN_TC_GDEPTH=4"
V[tc25]="-DHECNN_TC_STAGES=2 -DHECNN_TC_GDEPTH=5"
V[nosacc]="-DHECNN_KS_ABLATE_SACC"
V[b12e4]="-DHECNN_KS_LOGB=12 -DHECNN_KS_LOGE=4 -DHECNN_KS_MAXT_COL=256 -DHECNN_KS_MINB=2"
for name in "${!V[@]}"; do
  [ -n "$1" ] && [[ ! " $* " =~ " $name " ]] && continue
  make -s -C paper_1911_11377_b200/csrc -j8 OUT=$PWD/build_variants/$name OBJ=$PWD/build_variants/$name/obj EXTRA_NVFLAGS="${V[$name]}" >/dev/null
  echo "built $name: ${V[$name]}"
done
