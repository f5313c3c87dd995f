#!/bin/bash
# Runs the NTT micro-benchmark and a short bench for every library variant in build_variants/.
for so in build_variants/*.so; do
  tag=$(basename $so .so)
  echo "== $tag"
  HENET_B200_LIB=$PWD/$so python scripts/ntt_micro.py 2>&1 | grep -E "fwd|inv"
  HENET_B200_LIB=$PWD/$so python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$tag.json 2>/dev/null
  python scripts/show_bench.py gpurun_out/bench_$tag.json 2>/dev/null | grep -E "^value|k_relin|k_rescale|k_ntt"
done
