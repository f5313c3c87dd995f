# GPU-box A/B of library variants in build_variants/: optional quick parity subset, then a short
# bench per variant (device-resident step only).
# usage: bash scripts/gpu/ab.sh TAG "kernel regex" ["pytest -k expr"]
TAG=${1:-ab}
PAT=${2:-keysw}
K=${3:-}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for so in build_variants/*.so; do
  v=$(basename $so .so)
  if [ -n "$K" ]; then
    HENET_B200_LIB=$PWD/$so timeout 600 python -m pytest tests -m gpu -q -p no:cacheprovider -k "$K" > gpurun_out/${TAG}_${v}_tests.log 2>&1
    echo "== $v tests rc=$? $(tail -1 gpurun_out/${TAG}_${v}_tests.log)"
  fi
  HENET_B200_LIB=$PWD/$so timeout 300 python bench.py --steps 10 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_${v}.json 2>/dev/null
  echo "== $v"; python scripts/show_bench.py gpurun_out/${TAG}_${v}.json 2>/dev/null | grep -E "^value|$PAT"
done
