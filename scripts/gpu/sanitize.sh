# GPU-box: compute-sanitizer tools over the parity tests that cover the TMEM (tcgen05.alloc /
# ld / st), mbarrier, cp.async and cp.async.bulk kernels at toy sizes, plus the wide tensor-core
# contraction and the client kernels (encrypt / decrypt / refresh).
# usage: bash scripts/gpu/sanitize.sh TAG tool [tool ...]   (memcheck racecheck synccheck initcheck)
TAG=${1:-san}
shift
TOOLS=${@:-memcheck}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
SEL="relin_levels or rescale_levels or tensor_core or dense_and_conv or ntt_every_prime or execute_toy_bit_exact or square_relin_rescale or dense_c5b_shape_small or conv_c4_shape_small or wide_relinearize or encrypt_tensor_bit_exact or refresh_engine_bit_exact or decrypt_residues"
for TOOL in $TOOLS; do
  EXTRA=()
  [ "$TOOL" = "racecheck" ] && EXTRA=(--racecheck-report all)
  timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool "$TOOL" "${EXTRA[@]}" --target-processes all --print-limit 50 \
    --log-file gpurun_out/${TAG}_${TOOL}.log \
    python -m pytest tests/test_gpu_vs_oracle.py tests/test_gpu_parity.py tests/test_gpu_wide.py tests/test_gpu_client.py \
    -m gpu -q -p no:cacheprovider -k "$SEL" \
    > gpurun_out/${TAG}_${TOOL}_pytest.log 2>&1
  echo "$TOOL rc=$?"
  tail -3 gpurun_out/${TAG}_${TOOL}_pytest.log
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY" gpurun_out/${TAG}_${TOOL}.log | sort | uniq -c | head -10
done
