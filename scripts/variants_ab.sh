#!/bin/bash
# Short bench of every library variant in build_variants/ (A/B runs); prints the kernels named by $1.
pat=${1:-conv}
for so in build_variants/*.so; do
  tag=$(basename $so .so)
  HENET_B200_LIB=$PWD/$so python bench.py --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/bench_$tag.json 2>/dev/null
  echo "== $tag"; python scripts/show_bench.py gpurun_out/bench_$tag.json 2>/dev/null | grep -E "^value|$pat"
done
