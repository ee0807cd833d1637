#!/bin/bash
# Build cellbench against kernel-source variants (-D flags) and run each (development).
#   tools/cellbench/run.sh build "name:-DFOO=1,-DBAR=2" ...   (here, no GPU needed)
#   tools/cellbench/run.sh run                                  (on the GPU box)
set -e
cd "$(dirname "$0")/../.."
OUT=variants/cellbench
if [ "$1" = build ]; then
  shift
  mkdir -p $OUT build/cellbench
  for spec in "$@"; do
    name=${spec%%:*}; defs=$(echo "${spec#*:}" | tr ',' ' ')
    objs=""
    for f in paper_1509_04232_b200/csrc/*.cu tools/cellbench/cellbench.cu; do
      o=build/cellbench/${name}_$(basename $f).o
      nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Iinclude $defs -c $f -o $o &
      objs="$objs $o"
    done
    wait
    nvcc -gencode arch=compute_100a,code=sm_100a -o $OUT/cellbench_$name $objs
    echo built $OUT/cellbench_$name
  done
else
  for b in $OUT/cellbench_*; do echo "== $(basename $b)"; timeout 120 $b ${@:2}; done
fi
