#!/usr/bin/env bash
# Build A/B variants of the product library with extra -D switches (CPU side):
#   scripts/ab_variants.sh build NAME "-DFOO=1 -DBAR=0" [NAME2 "..."]...
# Time them on the GPU box, alternating, through PSG_LIB (gpurun side):
#   scripts/ab_variants.sh run "<profile_step.py args>" NAME NAME2 ...   (base = product lib)
set -euo pipefail
ROOT=$(cd "$(dirname "$0")/.." && pwd)
cmd=$1; shift
if [ "$cmd" = build ]; then
  while [ $# -gt 0 ]; do
    name=$1; flags=$2; shift 2
    make -s -C "$ROOT/paper_2412_03451_b200/csrc" -j8 OBJ="/tmp/psg_variants/$name" \
      OUT="$ROOT/_variants/libpsplat_b200_$name.so" \
      NVFLAGS="-O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -gencode arch=compute_100a,code=sm_100a $flags"
    echo "built $name ($flags)"
  done
elif [ "$cmd" = run ]; then
  args=$1; shift
  for rep in 1 2; do
    for name in base "$@"; do
      if [ "$name" = base ]; then lib="$ROOT/paper_2412_03451_b200/lib/libpsplat_b200.so";
      else lib="$ROOT/_variants/libpsplat_b200_$name.so"; fi
      echo "== $name rep $rep"
      PSG_LIB=$lib python "$ROOT/scripts/profile_step.py" $args 2>&1 | grep -E "rep [1-9]|Error" | sed "s/, stats.*//; s/^/[$name] /"
    done
  done
fi
