# GPU-box: the whole -m gpu suite on the self-check build (HG_DEBUG_CHECKS=1: mbarrier waits
# trap after 2^24 polls instead of hanging, TMEM allocations are range-checked), the stand-in
# for compute-sanitizer, which is closed on this pool.
# usage: bash scripts/gpu/debug_checks.sh TAG   (build_debug/libhenet_b200.so built beforehand)
TAG=${1:-dbg}
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
HENET_B200_LIB=$PWD/build_debug/libhenet_b200.so timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider \
  > gpurun_out/${TAG}_debug_checks.log 2>&1
echo "pytest rc=$?"
grep -c "hg debug" gpurun_out/${TAG}_debug_checks.log
tail -3 gpurun_out/${TAG}_debug_checks.log
