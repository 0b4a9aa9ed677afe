#!/bin/bash
# build_variant.sh OUT.so SRC.cu [-DFLAGS...]: libwm_b200 with one source
# recompiled under extra flags (A/B kernel experiments; build/variants/).
set -e
out=$1; src=$2; shift 2
root=$(cd "$(dirname "$0")/.." && pwd)
objs=""
for f in wm_api wm_clique wm_motif wm_ingest wm_dict; do
  if [ "$f.cu" = "$src" ]; then
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
      -Xcompiler -fPIC,-O3 -Xptxas -O3 -I "$root/include" "$@" -c -o "$out.$f.o" \
      "$root/paper_2212_04551_b200/csrc/$src"
    objs="$objs $out.$f.o"
  else
    objs="$objs $root/build/obj/$f.o"
  fi
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out" $objs
rm -f "$out".*.o
