# GPU-box: one compute-sanitizer tool over the parity tests that cover the TMEM (tcgen05.alloc /
# ld / st), mbarrier, cp.async and cp.async.bulk kernels at toy sizes.
# usage: bash scripts/gpu/sanitize.sh memcheck|racecheck|synccheck|initcheck TAG
TOOL=${1:-memcheck}
TAG=${2:-san}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
SEL="relin_levels or rescale_levels or tensor_core or dense_and_conv or ntt_every_prime or execute_toy_bit_exact or square_relin_rescale"
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool "$TOOL" --target-processes all --print-limit 50 \
  --log-file gpurun_out/${TAG}_${TOOL}.log \
  python -m pytest tests/test_gpu_vs_oracle.py tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "$SEL" \
  > gpurun_out/${TAG}_${TOOL}_pytest.log 2>&1
echo "rc=$?"
tail -5 gpurun_out/${TAG}_${TOOL}_pytest.log
grep -E "ERROR SUMMARY|Error|error" gpurun_out/${TAG}_${TOOL}.log | sort | uniq -c | head -20
