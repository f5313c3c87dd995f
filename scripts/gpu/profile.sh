# GPU-box: bench + launch list + one ncu --set full capture of the step's kernels.
# usage: bash scripts/gpu/profile.sh TAG [kernel-regex] [extra bench args]
TAG=${1:-prof}
KRE=${2:-"regex:k_(relin|mac|rescale)"}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 600 python bench.py ${3} > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
tail -c 600 gpurun_out/${TAG}_bench.json
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python scripts/ncu_target.py > gpurun_out/${TAG}_launches.log 2>&1; echo "launches rc=$?"
NCU_STEPS=1 timeout 1500 $NCU --set full --import-source on --clock-control none -k "$KRE" -c 12 \
  -o gpurun_out/${TAG} python scripts/ncu_target.py > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/${TAG}_ncu.log
