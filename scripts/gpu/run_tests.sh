# GPU-box: a subset of the -m gpu suite (pytest -k expr) and the drop-in binary.
# usage: bash scripts/gpu/run_tests.sh TAG "pytest -k expr" [dropin]
TAG=${1:-t}
K=${2:-}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
if [ -n "$K" ]; then KARG=(-k "$K"); else KARG=(); fi
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 "${KARG[@]}" > gpurun_out/${TAG}_gputests.log 2>&1
echo "pytest rc=$?"
tail -60 gpurun_out/${TAG}_gputests.log
if [ "$3" = "dropin" ]; then
  timeout 900 oracle/_ref/dropin_test > gpurun_out/${TAG}_dropin.log 2>&1; echo "dropin rc=$?"; cat gpurun_out/${TAG}_dropin.log
  timeout 300 oracle/_ref/dropin_test --bench 10 > gpurun_out/${TAG}_dropin_bench.json 2>&1; cat gpurun_out/${TAG}_dropin_bench.json
fi
