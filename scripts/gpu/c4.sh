# GPU-box: c4 parity tests (conv geometries incl. 1x1, wide block, stated shape, fallbacks) and
# the c4 bench with per-node and refresh-engine traces.
# usage: bash scripts/gpu/c4.sh TAG [extra env for the diagnostic rerun]
TAG=${1:-c4}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_conv.py tests/test_gpu_wide.py tests/test_gpu_stated_shapes.py tests/test_gpu_fallbacks.py -m gpu -q -p no:cacheprovider -x > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?"; tail -5 gpurun_out/${TAG}_tests.log
HG_NODE_TIMING=1 HG_REFRESH_TRACE=1 timeout 900 python bench.py --workload c4 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_c4.json 2> gpurun_out/${TAG}_bench_c4.err
echo "c4 bench rc=$?"; python -c "import json,sys; d=json.load(open(sys.argv[1])); print(d['value'], d['tile_ms'], d['tile_ms_steps'], d['clocks'])" gpurun_out/${TAG}_bench_c4.json; grep -E "c4 step|refresh layer" gpurun_out/${TAG}_bench_c4.err | cut -c1-400
HG_BENCH_NO_CLOCKS=1 HG_NODE_TIMING=1 HG_REFRESH_TRACE=1 timeout 900 python bench.py --workload c4 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_c4_noclk.json 2> gpurun_out/${TAG}_bench_c4_noclk.err
echo "c4 bench (no clock sampler) rc=$?"; python -c "import json,sys; d=json.load(open(sys.argv[1])); print(d['value'], d['tile_ms'], d['tile_ms_steps'])" gpurun_out/${TAG}_bench_c4_noclk.json; grep -E "c4 step|refresh layer" gpurun_out/${TAG}_bench_c4_noclk.err | cut -c1-400
