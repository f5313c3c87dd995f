#!/bin/bash
# Builds library variants for GPU A/B runs: scripts/build_variants.sh name1:"-DX=1 -DY=0" name2:"" ...
# Each variant gets its own object directory under /tmp and lands in build_variants/<name>.so.
mkdir -p build_variants
pids=()
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  ( make -s -C paper_1908_04172_b200/csrc -j4 OUT=$PWD/build_variants/$name.so BUILD=/tmp/hg_build_$name HGDEFS="$defs" \
      > /tmp/hg_build_$name.log 2>&1 && echo "built $name" || { echo "FAILED $name"; tail -20 /tmp/hg_build_$name.log; } ) &
  pids+=($!)
done
wait "${pids[@]}"
