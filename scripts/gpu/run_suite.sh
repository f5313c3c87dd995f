# GPU-box driver for one gpurun call: the -m gpu suite, the drop-in e2e timing and the bench.
# usage: bash scripts/gpu/run_suite.sh TAG [pytest -k expr]
TAG=${1:-run}
K=${2:-}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
{ nproc; free -g | head -2; lscpu | grep "Model name"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; } > gpurun_out/${TAG}_host.txt 2>&1
if [ -n "$K" ]; then KARG=(-k "$K"); else KARG=(); fi
timeout 2700 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=30 "${KARG[@]}" > gpurun_out/${TAG}_gputests.log 2>&1
echo "pytest rc=$?"
tail -45 gpurun_out/${TAG}_gputests.log
timeout 300 oracle/_ref/dropin_test --bench 10 > gpurun_out/${TAG}_dropin_bench.json 2>&1; cat gpurun_out/${TAG}_dropin_bench.json
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/${TAG}_bench.json
