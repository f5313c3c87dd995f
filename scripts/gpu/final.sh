# GPU-box: the round's final evidence run -- smoke(), the whole -m gpu suite, the drop-in binary
# and its e2e timing, the default bench line (c2), the other BASELINE configs, the reference arm,
# and the launch list + ncu --set full of the c2 step's kernels.
# usage: bash scripts/gpu/final.sh TAG
TAG=${1:-final}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
{ nproc; lscpu | grep "Model name"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; } > gpurun_out/${TAG}_host.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/${TAG}_gputests.log 2>&1
echo "pytest rc=$?"; grep -E "passed|failed" gpurun_out/${TAG}_gputests.log | tail -1
timeout 900 oracle/_ref/dropin_test > gpurun_out/${TAG}_dropin.log 2>&1; echo "dropin rc=$?"
timeout 300 oracle/_ref/dropin_test --bench 10 > gpurun_out/${TAG}_dropin_bench.json 2>&1; head -1 gpurun_out/${TAG}_dropin_bench.json
timeout 600 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
for w in c1 c3 c4 c5b; do timeout 900 python bench.py --workload $w > gpurun_out/${TAG}_bench_$w.json 2> gpurun_out/${TAG}_bench_$w.err; echo "bench $w rc=$?"; done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err; echo "ref rc=$?"
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python scripts/ncu_target.py > gpurun_out/${TAG}_launches.log 2>&1; echo "launches rc=$?"
NCU_STEPS=1 timeout 1500 $NCU --set full --import-source on --clock-control none -k "regex:k_(relin|mac|rescale)" -c 12 \
  -o gpurun_out/${TAG}_prof python scripts/ncu_target.py > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
