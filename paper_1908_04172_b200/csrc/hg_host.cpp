// SPDX-License-Identifier: Apache-2.0
//
// Host runtime + C ABI (include/henet_b200.h).  Everything numerical runs in
// the sm_100a kernels of hg_kernels.cu; this file owns parameters, tables,
// scale/level bookkeeping (bit-identical double arithmetic to the reference),
// validation with the reference's error messages, device memory, the model
// and plan objects, and the graph executor.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <functional>
#include <mutex>
#include <set>

#include "hg_modmath.hpp"
#include "hg_runtime.hpp"

namespace hg {

namespace {
thread_local std::string g_last_error;

template <class F>
int guard(F&& f) {
  try {
    f();
    return HG_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "allocation failed";
    return HG_ERR_ALLOC;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return HG_ERR_INTERNAL;
  }
}
}  // namespace

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    throw Error(e == cudaErrorMemoryAllocation ? HG_ERR_ALLOC : HG_ERR_CUDA,
                std::string(what) + ": " + cudaGetErrorString(e));
  }
}

static void check_launch(int r, const char* what) {
  if (r < 0) throw Error(HG_ERR_UNSUPPORTED, std::string(what) + ": unsupported configuration");
  cuda_check(cudaGetLastError(), what);
}

// Buffers of at least 1 MB (HG_BUF_CACHE_MIN_MB) released on the context's stream are recycled
// by exact size (DeviceCore::take / put) instead of going back to the driver's pool.  The
// threshold was 1 GiB (c4 / c5b layers only) until the two-batches-in-flight schedule showed
// cudaMallocAsync itself stalling: with two contexts executing concurrently, the second
// execute on a context after a device synchronise spent 2-3 ms in its layer-sized allocations
// every time and 10-500 ms in about one run in five, whatever the pool (device default or
// per context), the auxiliary stream or the kernel parameter size (profiles/r3_experiments.md).
static const size_t kBufCacheMin = [] {
  const char* e = getenv("HG_BUF_CACHE_MIN_MB");
  return e ? static_cast<size_t>(atof(e) * 1048576.0) : (size_t(1) << 20);
}();
static size_t buf_cache_max(int device) {
  static std::mutex mu;
  static std::map<int, size_t> v;
  std::lock_guard<std::mutex> g(mu);
  auto it = v.find(device);
  if (it != v.end()) return it->second;
  size_t cap = 0;
  const char* off = getenv("HG_BUF_CACHE");
  if (!(off != nullptr && off[0] == '0')) {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) == cudaSuccess) cap = tot / 2;  // default: half the device
    if (const char* e = getenv("HG_BUF_CACHE_MAX_GB")) cap = static_cast<size_t>(atof(e) * 1073741824.0);
  }
  v[device] = cap;
  return cap;
}

// Every context on a device has its own cache; the cap (half the device by default) bounds
// their sum, and an allocation that fails releases all of them before it is retried.
namespace {
std::mutex g_cores_mu;
std::map<int, std::set<DeviceCore*>> g_cores;   // live cores per device
std::map<int, size_t> g_cached_total;           // bytes held by their caches
}  // namespace

void DeviceCore::enroll() {
  std::lock_guard<std::mutex> g(g_cores_mu);
  g_cores[device].insert(this);
}

// Lock order: g_cores_mu, then a core's cache_mu.
void* DeviceCore::take(size_t bytes) {
  std::lock_guard<std::mutex> gt(g_cores_mu);
  std::lock_guard<std::mutex> g(cache_mu);
  auto it = cache.find(bytes);
  if (it == cache.end()) return nullptr;
  void* p = it->second;
  cache.erase(it);
  cached -= bytes;
  g_cached_total[device] -= bytes;
  return p;
}

bool DeviceCore::put(void* p, size_t bytes) {
  const size_t cap = buf_cache_max(device);
  std::lock_guard<std::mutex> gt(g_cores_mu);
  std::lock_guard<std::mutex> g(cache_mu);
  if (g_cached_total[device] + bytes > cap) return false;
  g_cached_total[device] += bytes;
  cache.emplace(bytes, p);
  cached += bytes;
  return true;
}

// g_cores_mu held
static void flush_core_locked(DeviceCore* c) {
  std::lock_guard<std::mutex> g(c->cache_mu);
  for (auto& e : c->cache) cudaFreeAsync(e.second, c->stream);
  c->cache.clear();
  g_cached_total[c->device] -= c->cached;
  c->cached = 0;
}

void DeviceCore::flush() {
  std::lock_guard<std::mutex> gt(g_cores_mu);
  flush_core_locked(this);
}

// Releases the caches of every context on the device and waits for the frees (out-of-memory path).
static void flush_device_caches(int device) {
  std::lock_guard<std::mutex> gt(g_cores_mu);
  for (DeviceCore* c : g_cores[device]) {
    flush_core_locked(c);
    cudaStreamSynchronize(c->stream);
  }
}

DeviceCore::~DeviceCore() {
  {
    std::lock_guard<std::mutex> g(g_cores_mu);
    g_cores[device].erase(this);
  }
  if (stream) {
    cudaSetDevice(device);
    flush();
    cudaStreamSynchronize(stream);
    cudaStreamDestroy(stream);
  }
}

DeviceBuffer::DeviceBuffer(std::shared_ptr<DeviceCore> c, size_t b, cudaStream_t s) : core(std::move(c)), bytes(b) {
  stream = s ? s : core->stream;
  if (bytes == 0) return;
  const bool cacheable = bytes >= kBufCacheMin && stream == core->stream;
  if (cacheable && (ptr = core->take(bytes)) != nullptr) return;
  cudaError_t e = cudaMallocAsync(&ptr, bytes, stream);
  if (e == cudaErrorMemoryAllocation) {
    // the caches (this context's or another's on the device) may hold the memory: release
    // them (stream-ordered) and retry once
    cudaGetLastError();
    flush_device_caches(core->device);
    e = cudaMallocAsync(&ptr, bytes, stream);
  }
  cuda_check(e, "cudaMallocAsync");
}

DeviceBuffer::~DeviceBuffer() {
  if (!ptr) return;
  if (bytes >= kBufCacheMin && stream == core->stream && core->put(ptr, bytes)) return;
  cudaFreeAsync(ptr, stream);
}

// ---------------------------------------------------------------------------
// Context (henet/params.hpp:112-129)
// ---------------------------------------------------------------------------
static std::shared_ptr<Context> make_context(u32 n, const u64* chain, u32 chain_len, u64 special, double scale,
                                             int device) {
  require(n >= 2 && (n & (n - 1)) == 0, "poly degree must be a power of two");
  require(chain_len >= 1, "modulus chain must be non-empty");
  u32 logn = 0;
  while ((1u << logn) < n) ++logn;
  if (logn < 11 || logn > 14 || (1u << logn) != n)
    throw Error(HG_ERR_UNSUPPORTED, "B200 kernels implement ring degrees 2^11..2^14 (got " + std::to_string(n) + ")");
  const u32 full = chain_len + (special ? 1 : 0);
  if (full > static_cast<u32>(kMaxPrimes)) throw Error(HG_ERR_UNSUPPORTED, "too many basis moduli");

  auto ctx = std::make_shared<Context>();
  ctx->n = n;
  ctx->logn = logn;
  ctx->chain.assign(chain, chain + chain_len);
  ctx->special = special;
  ctx->has_special = special != 0;
  ctx->default_scale = scale;
  for (u32 i = 0; i < full; ++i) {
    const u64 q = ctx->basis_mod(i);
    require(q >= 2, "modulus must be at least 2");
    require(nt::is_prime(q), "modulus must be prime");
    // u64 residues with lazy values in [0, 4q) (hg_wide.cuh): any prime below 2^62
    if (q >= (1ull << 62))
      throw Error(HG_ERR_UNSUPPORTED, "B200 kernels implement primes below 2^62 (got " + std::to_string(q) + ")");
    if (q >= (1ull << 30)) ctx->wide = true;
    for (u32 j = 0; j < i; ++j) {
      if (ctx->basis_mod(j) == q) {
        throw Error(HG_ERR_VALIDATION, i == chain_len ? "special prime must differ from the chain"
                                                      : "chain moduli must be pairwise distinct");
      }
    }
    if ((q - 1) % (2ull * n) != 0) throw Error(HG_ERR_VALIDATION, "modulus admits no 2N-th root of unity (q != 1 mod 2N)");
  }
  // N = 2^11 (preset P11) runs on the u64 kernels whatever its primes: the u32 kernels keep
  // per-thread rows in tensor memory, which needs CTAs of >= 128 threads (N >= 2^12).
  if (logn < 12) ctx->wide = true;
  long double acc = 1.0L;
  ctx->modulus_products.push_back(acc);
  for (u64 q : ctx->chain) {
    acc *= static_cast<long double>(q);
    ctx->modulus_products.push_back(acc);
  }

  int ndev = 0;
  cuda_check(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  require(device >= 0 && device < ndev, "no such CUDA device");
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  cudaDeviceProp prop{};
  cuda_check(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
  if (prop.major != 10) throw Error(HG_ERR_CUDA, "kernels are built for sm_100a; device is sm_" +
                                                     std::to_string(prop.major) + std::to_string(prop.minor));
  {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  {
    // Dot on the int8 tensor cores by default; HG_DENSE_TC=0 selects the IMAD kernel
    const char* tc = getenv("HG_DENSE_TC");
    ctx->dense_tc = !(tc != nullptr && tc[0] == '0');
  }
  ctx->core = std::make_shared<DeviceCore>();
  ctx->core->device = device;
  cuda_check(cudaStreamCreateWithFlags(&ctx->core->stream, cudaStreamNonBlocking), "cudaStreamCreate");
  ctx->core->enroll();

  // NTT tables (root_powers / inv_root_powers in the reference's order, with
  // Shoup companions), staged per NTT pass in the order the kernels consume them.
  const u32 LOGT = logn - 5, CB = logn >= 14 ? logn - 10 : 3, MB = LOGT - CB;
  const u32 rowsB = 1u << MB, rowsT = 1u << LOGT;
  const u32 FC = 1u << CB;  // pass-C scale factors per thread (Ntt::scale_C)
  const size_t per_prime = 2 * (static_cast<size_t>(rowsB) * 32 + static_cast<size_t>(rowsT) * FC);
  std::vector<uint2> staged(static_cast<size_t>(full) * per_prime);
  auto jmapB = [&](u32 tid, u32 k) -> u32 {
    const u32 CBm = (1u << CB) - 1, MBm = (1u << MB) - 1;
    return (tid & CBm) | ((k & MBm) << CB) | ((tid >> CB) << LOGT) | ((k >> MB) << (LOGT + MB));
  };
  // pass-B rows in the order the unrolled stages consume them (Ntt::fwd_pass / inv_pass)
  auto stage_rowsB = [&](bool inverse, const std::vector<uint2>& tab, uint2* out) {
    const u32 NB = MB, BLO = CB;
    for (u32 R = 0; R < rowsB; ++R) {
      const u32 tid = R << CB;
      int nslot = 0;
      for (u32 st = 0; st < NB; ++st) {
        const u32 rb = inverse ? st : NB - 1 - st;
        const u32 bb = BLO + rb;
        nslot = (nslot + 1) & ~1;  // stages start at even slots (Ntt::fwd_pass / inv_pass)
        for (u32 gg = 0; gg < (1u << (5 - NB)); ++gg)
          for (u32 hi = 0; hi < (1u << (NB - 1 - rb)); ++hi) {
            const u32 kh = (gg << NB) | (hi << (rb + 1));
            const u32 j = jmapB(tid, kh);
            out[static_cast<size_t>(R) * 32 + nslot++] = tab[(1u << (logn - 1 - bb)) + (j >> (bb + 1))];
          }
      }
    }
  };
  // pass C: psi^bitrev(idx) = V(b, c, g) * T_b(tid) over disjoint bit fields of idx
  auto stage_C = [&](bool inverse, u64 root, u64 q, uint2* vtab, uint2* tbase) {
    const u32 NB = CB;
    int nslot = 0;
    for (u32 st = 0; st < NB; ++st) {
      const u32 rb = inverse ? st : NB - 1 - st;
      const u32 bb = rb;
      const u32 nb = logn - 1 - bb;
      for (u32 gg = 0; gg < (1u << (5 - NB)); ++gg)
        for (u32 hi = 0; hi < (1u << (NB - 1 - rb)); ++hi) {
          const u32 u = hi | (gg << (CB + LOGT - bb - 1));
          const u64 v = nt::powmod(root, nt::bit_reverse((1u << nb) | u, logn), q);
          vtab[nslot++] = make_uint2(static_cast<u32>(v), nt::shoup(v, q));
        }
    }
    for (u32 t = 0; t < rowsT; ++t)
      for (u32 k = 0; k < FC; ++k) {
        u64 v = 1;  // F_k(t) = prod over the set bits b of k of T_b(t)
        for (u32 bb = 0; bb < CB; ++bb)
          if ((k >> bb) & 1) v = nt::mulmod(v, nt::powmod(root, nt::bit_reverse(t << (CB - bb - 1), logn), q), q);
        tbase[static_cast<size_t>(t) * FC + k] = make_uint2(static_cast<u32>(v), nt::shoup(v, q));
      }
  };
  std::vector<uint2> f(n), g(n);
  for (u32 i = 0; i < full; ++i) {
    const u64 q = ctx->basis_mod(i);
    const u64 psi = nt::primitive_2n_root(q, n);
    require(nt::powmod(psi, n, q) == q - 1 && nt::powmod(psi, 2ull * n, q) == 1, "root order check failed");
    ctx->roots.push_back(psi);
    const u64 psi_inv = nt::inv(psi, q);
    for (u32 k = 0; k < n; ++k) {
      const u32 rev = nt::bit_reverse(k, logn);
      const u64 w = nt::powmod(psi, rev, q), wi = nt::powmod(psi_inv, rev, q);
      f[k] = make_uint2(static_cast<u32>(w), nt::shoup(w, q));
      g[k] = make_uint2(static_cast<u32>(wi), nt::shoup(wi, q));
    }
    DevPrime& P = ctx->basis.p[i];
    P.q = static_cast<u32>(q);
    P.two_q = static_cast<u32>(2 * q);
    P.half = static_cast<u32>(q >> 1);
    P.mu32 = static_cast<u32>((1ull << 32) / q);
    P.mu64 = static_cast<u64>((static_cast<nt::u128>(1) << 64) / q);
    P.r32 = static_cast<u32>((1ull << 32) % q);
    {
      u32 k = 0;
      while ((1ull << k) <= q) ++k;  // bit length
      P.bsh = k - 1;
      P.bmu = static_cast<u32>((static_cast<nt::u128>(1) << (k + 31)) / q);
    }
    const u64 ninv = nt::inv(n % q, q);
    P.ninv = static_cast<u32>(ninv);
    P.ninv_sh = nt::shoup(ninv, q);
    const u64 w1n = nt::mulmod(g[1].x, ninv, q);
    P.w1n = static_cast<u32>(w1n);
    P.w1n_sh = nt::shoup(w1n, q);
    for (u32 k = 0; k < 32; ++k) {
      P.twA[k] = f[k];
      P.itwA[k] = g[k];
    }
    uint2* base = &staged[static_cast<size_t>(i) * per_prime];
    stage_rowsB(false, f, base);
    stage_C(false, psi, q, P.tvC, base + rowsB * 32);
    stage_rowsB(true, g, base + rowsB * 32 + rowsT * FC);
    stage_C(true, psi_inv, q, P.itvC, base + 2 * rowsB * 32 + rowsT * FC);
  }
  if (ctx->wide) {
    // u64 path: natural-order tables with 64-bit Shoup companions (hg_wide.cuh)
    std::vector<ulonglong2> tw(static_cast<size_t>(full) * 2 * n);
    for (u32 i = 0; i < full; ++i) {
      const u64 q = ctx->basis_mod(i);
      const u64 psi = ctx->roots[i], psi_inv = nt::inv(psi, q);
      auto sh64 = [&](u64 w) { return static_cast<u64>((static_cast<nt::u128>(w) << 64) / q); };
      ulonglong2* fw = &tw[static_cast<size_t>(i) * 2 * n];
      ulonglong2* iw = fw + n;
      for (u32 k = 0; k < n; ++k) {
        const u32 rev = nt::bit_reverse(k, logn);
        const u64 w = nt::powmod(psi, rev, q), wi = nt::powmod(psi_inv, rev, q);
        fw[k] = make_ulonglong2(w, sh64(w));
        iw[k] = make_ulonglong2(wi, sh64(wi));
      }
      DevPrimeW& W = ctx->basisw.p[i];
      W.q = q;
      W.two_q = 2 * q;
      W.half = q >> 1;
      const u64 d1 = static_cast<u64>((static_cast<nt::u128>(1) << 64) / q);
      const u64 r1 = static_cast<u64>((static_cast<nt::u128>(1) << 64) % q);
      W.r128_hi = d1;
      W.r128_lo = static_cast<u64>((static_cast<nt::u128>(r1) << 64) / q);
      const u64 ninv = nt::inv(n % q, q);
      W.ninv = ninv;
      W.ninv_sh = sh64(ninv);
      W.w1n = nt::mulmod(iw[1].x, ninv, q);
      W.w1n_sh = sh64(W.w1n);
      W.t64 = r1;
    }
    ctx->basisw.narrow = &ctx->basis;  // the u32 tables of the limbs below 2^30 (launch_ntt_w)
    ctx->wide_tables = ctx->alloc(tw.size() * sizeof(ulonglong2), nullptr);
    cuda_check(cudaMemcpyAsync(ctx->wide_tables->ptr, tw.data(), tw.size() * sizeof(ulonglong2),
                               cudaMemcpyHostToDevice, ctx->core->stream),
               "upload wide tables");
    for (u32 i = 0; i < full; ++i) {
      const ulonglong2* base = static_cast<const ulonglong2*>(ctx->wide_tables->ptr) + static_cast<size_t>(i) * 2 * n;
      ctx->basisw.p[i].fwd = base;
      ctx->basisw.p[i].inv = base + n;
    }
  }
  ctx->tables = ctx->alloc(staged.size() * sizeof(uint2), nullptr);
  cuda_check(cudaMemcpyAsync(ctx->tables->ptr, staged.data(), staged.size() * sizeof(uint2), cudaMemcpyHostToDevice,
                             ctx->core->stream),
             "upload tables");
  for (u32 i = 0; i < full; ++i) {
    const uint2* base = static_cast<const uint2*>(ctx->tables->ptr) + static_cast<size_t>(i) * per_prime;
    ctx->basis.p[i].fwdB = base;
    ctx->basis.p[i].fwdT = base + rowsB * 32;
    ctx->basis.p[i].invB = base + rowsB * 32 + rowsT * FC;
    ctx->basis.p[i].invT = base + 2 * rowsB * 32 + rowsT * FC;
  }
  cuda_check(cudaStreamSynchronize(ctx->core->stream), "upload tables");

  // Embedding tables, computed with the reference's expressions (henet/fft.hpp:30-43)
  // on the host libm so the GPU FFT sees identical doubles.
  const double pi = std::acos(-1.0);
  ctx->host_roots.resize(n);  // n/2 complex
  for (u32 k = 0; k < n / 2; ++k) {
    double ang = -2.0 * pi * k / n;
    ctx->host_roots[2 * k] = std::cos(ang);
    ctx->host_roots[2 * k + 1] = std::sin(ang);
  }
  ctx->host_twist.resize(2 * static_cast<size_t>(n));
  for (u32 k = 0; k < n; ++k) {
    double ang = pi * k / n;
    ctx->host_twist[2 * k] = std::cos(ang);
    ctx->host_twist[2 * k + 1] = std::sin(ang);
  }
  ctx->fft_tables = ctx->alloc((ctx->host_roots.size() + ctx->host_twist.size()) * sizeof(double), nullptr);
  cuda_check(cudaMemcpyAsync(ctx->fft_tables->ptr, ctx->host_roots.data(), ctx->host_roots.size() * sizeof(double),
                             cudaMemcpyHostToDevice, ctx->core->stream),
             "upload fft roots");
  cuda_check(cudaMemcpyAsync(static_cast<double*>(ctx->fft_tables->ptr) + ctx->host_roots.size(),
                             ctx->host_twist.data(), ctx->host_twist.size() * sizeof(double),
                             cudaMemcpyHostToDevice, ctx->core->stream),
             "upload fft twist");
  cuda_check(cudaStreamSynchronize(ctx->core->stream), "context init");
  return ctx;
}

// ---------------------------------------------------------------------------
// Helpers
// ---------------------------------------------------------------------------
static u32 inv_mod_u32(u64 a, u64 q) { return static_cast<u32>(nt::inv(a % q, q)); }

static void ensure(const Context& ctx, CtBatch& b, u64 count, u32 polys, u32 level, cudaStream_t s) {
  const u64 need = count * polys * level * static_cast<u64>(ctx.n) * ctx.word_bytes();
  if (!b.buf || b.buf->bytes < need || b.buf.use_count() > 1) b.buf = ctx.alloc(need, s);
  b.count = count;
  b.polys = polys;
  b.level = level;
}

static bool scales_match(double a, double b) { return std::fabs(a - b) / a <= std::ldexp(1.0, -40); }

// check_same_shape, henet/ckks.hpp:163-169
static void check_same_shape(const CtBatch& a, const CtBatch& b) {
  require(a.level == b.level, "ciphertext level mismatch");
  require(a.packing == b.packing, "packing mode mismatch");
  require(a.polys == b.polys, "ciphertext size mismatch");
  require(a.count == b.count, "element count mismatch");
  require(scales_match(a.scale, b.scale), "ciphertext scale mismatch");
}

// check_cc_mul, henet/ckks.hpp:396-401
static void check_cc_mul(const CtBatch& a) {
  require(a.packing == HG_PACKING_REAL, "ciphertext-ciphertext multiply is undefined under complex packing");
  require(a.polys == 2, "operands must be size-2 ciphertexts");
  require(a.level >= 1, "ciphertext exhausted");
}

// ---------------------------------------------------------------------------
// Device op building blocks (all asynchronous on stream s)
// ---------------------------------------------------------------------------
static void run_ew(const Context& ctx, EwArgs a, cudaStream_t s) {
  a.N = ctx.n;
  if (a.pt_div == 0) a.pt_div = 1;
  int r;
  if (ctx.wide) {
    // same argument block, u64 residues (the pointers address u64 buffers in wide mode)
    EwArgsW w{};
    w.op = a.op;
    w.a = reinterpret_cast<const u64*>(a.a);
    w.b = reinterpret_cast<const u64*>(a.b);
    w.res = reinterpret_cast<const u64*>(a.res);
    w.per_element = a.per_element;
    w.pt_div = a.pt_div;
    w.out = reinterpret_cast<u64*>(a.out);
    w.count = a.count;
    w.polys_a = a.polys_a;
    w.polys_out = a.polys_out;
    w.level = a.level;
    w.N = a.N;
    w.gidx = a.gidx;
    w.gw = a.gw;
    r = launch_elementwise_w(w, ctx.basisw, s);
  } else {
    r = launch_elementwise(a, ctx.basis, s);
  }
  check_launch(r, "elementwise");
}

// Encoded-residue buffers hold u32 or u64 words depending on the context mode.
static int encode_f32(const Context& ctx, const float* vals, u64 count, u32 row_len, u32 row_stride, u64 limb_stride,
                      u32 level, double scale, void* out, cudaStream_t s) {
  return ctx.wide ? launch_encode_scalars_w_f32(vals, count, row_len, row_stride, limb_stride, level, scale,
                                                static_cast<u64*>(out), ctx.basisw, s)
                  : launch_encode_scalars_f32(vals, count, row_len, row_stride, limb_stride, level, scale,
                                              static_cast<u32*>(out), ctx.basis, s);
}

// rescale_next applied (level - target) times; henet/ckks.hpp:504-519.
static CtBatch do_rescale(const Context& ctx, const CtBatch& in, u32 target, cudaStream_t s) {
  require(in.level >= 2, "cannot rescale below level 1");
  require(target >= 1 && target < in.level, "bad rescale target");
  CtBatch cur = in;
  while (cur.level > target) {
    const u32 L = cur.level;
    CtBatch out;
    out.packing = cur.packing;
    out.shape = cur.shape;
    ensure(ctx, out, cur.count, cur.polys, L - 1, s);
    const u64 p = ctx.chain[L - 1];
    int r;
    if (ctx.wide) {
      // Limbs with primes < 2^30 (all but the 40-bit limb 0 of the BASELINE wide chain) are
      // rescaled by the u32 kernel on a copy of their residues; the wide kernel then only
      // handles limb 0 (it repeats the dropped limb's inverse transform for its correction).
      bool hybrid = L >= 3 && p < (1ull << 30) && ctx.chain[0] >= (1ull << 30);
      for (u32 i = 1; hybrid && i + 1 < L; ++i) hybrid = ctx.chain[i] < (1ull << 30);
      static const bool wide_narrow = [] {
        const char* e = getenv("HG_WIDE_NARROW_RESCALE");
        return !(e != nullptr && e[0] == '0');
      }();
      hybrid = hybrid && wide_narrow;
      RescaleArgsW a{};
      a.in = cur.data64();
      a.out = out.data64();
      a.rows = cur.count * cur.polys;
      a.level = L;
      a.limb_cnt = hybrid ? 1 : 0;
      BufPtr corr64;
      if (p >= (1ull << 32)) {  // centred corrections beyond i32: a global row per polynomial
        corr64 = ctx.alloc(a.rows * ctx.n * sizeof(i64), s);
        a.corr64 = static_cast<i64*>(corr64->ptr);
      }
      for (u32 i = 0; i + 1 < L; ++i) {
        const u64 q = ctx.chain[i];
        a.pinv[i] = nt::inv(p % q, q);
        a.pinv_sh[i] = static_cast<u64>((static_cast<nt::u128>(a.pinv[i]) << 64) / q);
      }
      r = launch_rescale_w(static_cast<int>(ctx.logn), a, ctx.basisw, s);
      if (hybrid && r >= 0) {
        check_launch(r, "rescale (wide limb)");
        const u32 cnt = L - 1;  // limbs 1 .. L-1 (the dropped one last), in place in the u64 rows
        const u64 rows = cur.count * cur.polys;
        RescaleArgs na{};
        na.in64 = cur.data64();
        na.out64 = out.data64();
        na.io_level_in = L;
        na.io_level_out = L - 1;
        na.io_off = 1;
        na.rows = rows;
        na.level = cnt;
        na.lazy = 1;
        Basis sub{};
        for (u32 i = 0; i < cnt; ++i) sub.p[i] = ctx.basis.p[1 + i];
        for (u32 i = 0; i + 1 < cnt; ++i) {
          const u64 q = ctx.chain[1 + i];
          na.pinv[i] = inv_mod_u32(p, q);
          na.pinv_sh[i] = nt::shoup(na.pinv[i], q);
          na.pm[i] = static_cast<u32>((p / 2 + q - 1) / q * q);
          if (na.pm[i] + p / 2 >= 4 * q) na.lazy = 0;
        }
        r = launch_rescale(static_cast<int>(ctx.logn), na, sub, s);
      }
    } else {
      RescaleArgs a{};
      a.in = cur.data();
      a.out = out.data();
      a.rows = cur.count * cur.polys;
      a.level = L;
      a.lazy = 1;
      for (u32 i = 0; i + 1 < L; ++i) {
        const u64 q = ctx.chain[i];
        a.pinv[i] = inv_mod_u32(p, q);
        a.pinv_sh[i] = nt::shoup(a.pinv[i], q);
        a.pm[i] = static_cast<u32>((p / 2 + q - 1) / q * q);
        if (a.pm[i] + p / 2 >= 4 * q) a.lazy = 0;
      }
      r = launch_rescale(static_cast<int>(ctx.logn), a, ctx.basis, s);
    }
    check_launch(r, "rescale");
    out.scale = cur.scale / static_cast<double>(p);
    cur = std::move(out);
  }
  return cur;
}

// relinearize for u64 contexts (any primes < 2^62; presets P11-P14): the size-3 input is
// formed by the element-wise tensor kernel (square: a == b), then the three kernels of
// launch_relin_w, then an optional separate rescale.
static CtBatch do_relin_wide(const Context& ctx, const RelinKeyDev& rk, const CtBatch* a, const CtBatch* b, int mode,
                             bool rescale, cudaStream_t s) {
  const u32 L = a->level;
  const u32 n = ctx.n;
  if (rescale) require(L >= 2, "cannot rescale below level 1");
  CtBatch c3;
  const CtBatch* in3 = a;
  if (mode != 0) {
    c3.packing = a->packing;
    c3.shape = a->shape;
    c3.scale = a->scale * (b ? b->scale : a->scale);
    ensure(ctx, c3, a->count, 3, L, s);
    EwArgs e{};
    e.op = EwOp::Tensor;
    e.a = a->data();
    e.b = b ? b->data() : a->data();
    e.out = c3.data();
    e.count = a->count;
    e.polys_a = 2;
    e.polys_out = 3;
    e.level = L;
    run_ew(ctx, e, s);
    in3 = &c3;
  }
  CtBatch out;
  out.packing = a->packing;
  out.shape = a->shape;
  out.scale = in3->scale;
  ensure(ctx, out, a->count, 2, L, s);
  BufPtr D = ctx.alloc(a->count * L * static_cast<u64>(n) * 8, s);
  BufPtr ACC = ctx.alloc(a->count * 2 * (L + 1) * static_cast<u64>(n) * 8, s);
  BufPtr CORR = ctx.alloc(a->count * 2 * static_cast<u64>(n) * 8, s);
  RelinArgsW r{};
  r.A = in3->data64();
  r.out = out.data64();
  r.D = static_cast<u64*>(D->ptr);
  r.ACC = static_cast<u64*>(ACC->ptr);
  r.CORR = static_cast<i64*>(CORR->ptr);
  r.key = static_cast<const u64*>(rk.key->ptr);
  r.count = a->count;
  r.level = L;
  r.chain_len = static_cast<u32>(ctx.chain_len());
  for (u32 i = 0; i < L; ++i) {
    const u64 q = ctx.chain[i];
    r.pinvP[i] = nt::inv(ctx.special % q, q);
    r.pinvP_sh[i] = static_cast<u64>((static_cast<nt::u128>(r.pinvP[i]) << 64) / q);
  }
  check_launch(launch_relin_w(static_cast<int>(ctx.logn), r, ctx.basisw, s), "relinearize (wide)");
  if (!rescale) return out;
  return do_rescale(ctx, out, L - 1, s);
}

// relinearize(square / tensor / size-3) with optional fused rescale.
static CtBatch do_relin(const Context& ctx, const RelinKeyDev& rk, const CtBatch* a, const CtBatch* b, int mode,
                        bool rescale, cudaStream_t s) {
  require(ctx.has_special, "relinearization needs a special prime");
  require(rk.chain_len == ctx.chain_len(), "relinearization key has the wrong basis");
  if (ctx.wide) return do_relin_wide(ctx, rk, a, b, mode, rescale, s);
  const u32 L = a->level;
  const u32 n = ctx.n;
  if (rescale) require(L >= 2, "cannot rescale below level 1");
  // The merged mod-down + rescale feeds the rescale correction (|c| <= q_{L-1}/2) into the
  // lazy transform as c + q_i, which needs q_{L-1}/2 <= q_i for every kept limb; otherwise
  // (never for the BASELINE chains) relinearise, then rescale separately.
  bool fuse_rescale = rescale;
  for (u32 i = 0; rescale && i + 1 < L; ++i)
    if (ctx.chain[L - 1] / 2 > ctx.chain[i]) fuse_rescale = false;
  if (rescale && !fuse_rescale) {
    CtBatch r = do_relin(ctx, rk, a, b, mode, false, s);
    return do_rescale(ctx, r, L - 1, s);
  }
  CtBatch out;
  out.packing = a->packing;
  out.shape = a->shape;
  ensure(ctx, out, a->count, 2, rescale ? L - 1 : L, s);
  BufPtr D = ctx.alloc(a->count * L * static_cast<u64>(n) * 4, s);
  BufPtr ACC = ctx.alloc(a->count * 2 * L * static_cast<u64>(n) * 4, s);
  BufPtr CORR = ctx.alloc(a->count * 2 * static_cast<u64>(n) * 4, s);
  RelinArgs r{};
  r.A = a->data();
  r.Bm = b ? b->data() : a->data();
  r.mode = mode;
  r.count = a->count;
  r.level = L;
  r.chain_len = static_cast<u32>(ctx.chain_len());
  r.D = static_cast<u32*>(D->ptr);
  r.ACC = static_cast<u32*>(ACC->ptr);
  r.CORR = static_cast<i32*>(CORR->ptr);
  r.key = rk.key->ptr;
  r.out = out.data();
  r.rescale = rescale ? 1 : 0;
  for (u32 i = 0; i < L; ++i) {
    const u64 q = ctx.chain[i];
    r.pinvP[i] = inv_mod_u32(ctx.special, q);
    r.pinvP_sh[i] = nt::shoup(r.pinvP[i], q);
    r.pmP[i] = static_cast<u32>((ctx.special / 2 + q - 1) / q * q);
    if (rescale && i + 1 < L) {
      r.pinvL[i] = inv_mod_u32(ctx.chain[L - 1], q);
      r.pinvL_sh[i] = nt::shoup(r.pinvL[i], q);
    }
  }
  const int lr = launch_relin(static_cast<int>(ctx.logn), r, ctx.basis, s);
  check_launch(lr, "relinearize");
  // scale: square/mul_ct_ct multiply the scales; relinearize keeps it; rescale divides.
  double sc = a->scale;
  if (mode == 1) sc = a->scale * (b ? b->scale : a->scale);
  if (rescale) sc /= static_cast<double>(ctx.chain[L - 1]);
  out.scale = sc;
  return out;
}

static std::shared_ptr<CUevent_st> record_ready(cudaStream_t s) {
  cudaEvent_t ev;
  cuda_check(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
  cuda_check(cudaEventRecord(ev, s), "event");
  return std::shared_ptr<CUevent_st>(ev, [](cudaEvent_t e) { cudaEventDestroy(e); });
}

// Upload a float weight tensor once per model and device.  The copy is allocated on the
// context's stream (it outlives the caller's stream) and enqueued on `s`; executes on other
// streams wait on its ready event.  Caller holds the model mutex.
static const float* weight_dev(const Context& ctx, WeightTensor& w, cudaStream_t s) {
  auto it = w.dev.find(ctx.core.get());
  if (it != w.dev.end()) {
    cuda_check(cudaStreamWaitEvent(s, it->second.ready.get(), 0), "event");
    return static_cast<const float*>(it->second.buf->ptr);
  }
  KeptBuf k;
  k.buf = ctx.alloc(w.data.size() * sizeof(float), ctx.core->stream);
  if (s != ctx.core->stream) cuda_check(cudaStreamWaitEvent(s, record_ready(ctx.core->stream).get(), 0), "event");
  cuda_check(cudaMemcpyAsync(k.buf->ptr, w.data.data(), w.data.size() * sizeof(float), cudaMemcpyHostToDevice, s),
             "upload weights");
  k.ready = record_ready(s);
  w.dev[ctx.core.get()] = k;
  return static_cast<const float*>(k.buf->ptr);
}

// encode_scalar validation (henet/encoding.hpp:122-126, 180-188) for |value| <= max_abs.
static void check_scalar_encodable(const Context& ctx, double max_abs, u32 level, double scale) {
  require(level >= 1 && level <= ctx.chain_len(), "encode level out of range");
  require(scale > 0.0, "scale must be positive");
  const long double scaled = static_cast<long double>(max_abs) * static_cast<long double>(scale);
  require(scaled < ctx.modulus_products.at(level), "scaled magnitude exceeds q_level");
  require(std::fabs(static_cast<double>(scaled)) < std::ldexp(1.0, 100), "scaled magnitude too large to encode");
}

// encode_vector on the GPU: FFT encoder + NTT; returns device plaintexts [count][level][N].
// magnitude checks with the reference's long double arithmetic (henet/encoding.hpp:122-138)
static void check_magnitudes(const Context& ctx, u32 level, const unsigned long long* mant, const int* ex, u64 count) {
  for (u64 i = 0; i < count; ++i) {
    const long double mx = mant[i] ? std::ldexp(static_cast<long double>(mant[i]), ex[i]) : 0.0L;
    require(std::fabs(static_cast<double>(mx)) < std::ldexp(1.0, 100), "scaled magnitude too large to encode");
    require(mx < ctx.modulus_products.at(level) / 2.0L, "scaled magnitude exceeds q_level/2");
  }
}

// Deferred checks for chunked encoders: every chunk's per-vector maximum magnitudes stay on
// the device, and one read-back after the last chunk applies check_magnitudes (no host round
// trip per chunk).
struct DeferredMagnitudes {
  BufPtr buf;
  u64 count = 0;
  DeferredMagnitudes(const Context& c, u64 n, cudaStream_t s)
      : buf(c.alloc(n * (sizeof(unsigned long long) + sizeof(int)), s)), count(n) {}
  unsigned long long* mant(u64 e0) const { return static_cast<unsigned long long*>(buf->ptr) + e0; }
  int* ex(u64 e0) const { return reinterpret_cast<int*>(static_cast<unsigned long long*>(buf->ptr) + count) + e0; }
  void check(const Context& c, u32 level, cudaStream_t s) const {
    std::vector<unsigned long long> m(count);
    std::vector<int> e(count);
    cuda_check(cudaMemcpyAsync(m.data(), mant(0), count * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s), "d2h");
    cuda_check(cudaMemcpyAsync(e.data(), ex(0), count * sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
    cuda_check(cudaStreamSynchronize(s), "encode_vector");
    check_magnitudes(c, level, m.data(), e.data(), count);
  }
};

// defer != nullptr: the magnitudes go to defer at entry e0 and are checked later (no sync)
static BufPtr encode_vectors_dev(const Context& ctx, const double* d_slots, u32 n_slots, u64 count, u32 level,
                                 double scale, cudaStream_t s, std::vector<unsigned long long>& mant,
                                 std::vector<int>& ex, const DeferredMagnitudes* defer = nullptr, u64 e0 = 0) {
  require(level >= 1 && level <= ctx.chain_len(), "encode level out of range");
  require(scale > 0.0, "scale must be positive");
  require(n_slots <= ctx.n / 2, "more slots than the parameters provide");
  const u32 n = ctx.n;
  BufPtr out = ctx.alloc(count * level * static_cast<u64>(n) * ctx.word_bytes(), s);
  BufPtr scratch = ctx.alloc(count * static_cast<u64>(n) * sizeof(double2), s);
  BufPtr mags = ctx.alloc(count * static_cast<u64>(n) * sizeof(ulonglong2), s);
  BufPtr mm = defer ? nullptr : ctx.alloc(count * (sizeof(unsigned long long) + sizeof(int)), s);
  auto* d_mant = defer ? defer->mant(e0) : static_cast<unsigned long long*>(mm->ptr);
  auto* d_exp = defer ? defer->ex(e0) : reinterpret_cast<int*>(d_mant + count);
  const double2* roots = static_cast<const double2*>(ctx.fft_tables->ptr);
  const double2* twist = roots + n / 2;
  int r = launch_fft_encode(d_slots, n_slots, count, n, level, scale, roots, twist, static_cast<double2*>(scratch->ptr),
                            static_cast<ulonglong2*>(mags->ptr), d_mant, d_exp, s);
  check_launch(r, "fft encode");
  if (ctx.wide) {
    r = launch_pt_residues_ntt_w(static_cast<int>(ctx.logn), static_cast<const ulonglong2*>(mags->ptr), count, level,
                                 static_cast<u64*>(out->ptr), ctx.basisw, s);
    if (r == -2) {
      r = launch_mags_to_residues_w(static_cast<const ulonglong2*>(mags->ptr), count, n, level,
                                    static_cast<u64*>(out->ptr), ctx.basisw, s);
      check_launch(r, "residues");
      r = launch_ntt_w(static_cast<int>(ctx.logn), static_cast<u64*>(out->ptr), count * level, level, false,
                       ctx.basisw, s);
    }
  } else {
    r = launch_mags_to_residues(static_cast<const ulonglong2*>(mags->ptr), count, n, level,
                                static_cast<u32*>(out->ptr), ctx.basis, s);
    check_launch(r, "residues");
    r = launch_ntt(static_cast<int>(ctx.logn), static_cast<u32*>(out->ptr), count * level, level, false, ctx.basis, s);
  }
  check_launch(r, "ntt");
  if (defer) return out;
  mant.resize(count);
  ex.resize(count);
  cuda_check(cudaMemcpyAsync(mant.data(), d_mant, count * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s), "d2h");
  cuda_check(cudaMemcpyAsync(ex.data(), d_exp, count * sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
  cuda_check(cudaStreamSynchronize(s), "encode_vector");
  check_magnitudes(ctx, level, mant.data(), ex.data(), count);
  return out;
}

// ---------------------------------------------------------------------------
// Model: load_model's structural part (henet/graph.hpp:297-436)
// ---------------------------------------------------------------------------
static u64 elem_count(const std::vector<u32>& d) {
  u64 n = 1;
  for (u32 x : d) n *= x;
  return n;
}

static std::string shape_str(const std::vector<u32>& d) {
  std::string s = "(";
  for (size_t i = 0; i < d.size(); ++i) {
    if (i) s += ",";
    s += std::to_string(d[i]);
  }
  return s + ")";
}

static void finalize_model(Model& model) {
  require(!model.nodes.empty(), "manifest has no nodes");
  // topological sort, identical traversal order to the reference (stack of ready nodes)
  {
    std::map<std::string, std::vector<std::string>> fanout;
    std::map<std::string, size_t> indegree;
    for (const auto& n : model.nodes) indegree[n.id] = n.inputs.size();
    for (const auto& n : model.nodes) {
      for (const auto& in : n.inputs) {
        require(model.index.count(in), "node " + n.id + " references unknown input " + in);
        fanout[in].push_back(n.id);
      }
    }
    std::vector<Node> ordered;
    std::vector<std::string> ready;
    for (const auto& n : model.nodes)
      if (indegree[n.id] == 0) ready.push_back(n.id);
    while (!ready.empty()) {
      std::string id = ready.back();
      ready.pop_back();
      ordered.push_back(model.node(id));
      for (const auto& next : fanout[id])
        if (--indegree[next] == 0) ready.push_back(next);
    }
    require(ordered.size() == model.nodes.size(), "cycle detected in the graph");
    model.nodes = std::move(ordered);
    model.index.clear();
    for (size_t i = 0; i < model.nodes.size(); ++i) model.index[model.nodes[i].id] = i;
  }
  size_t inputs = 0, outputs = 0;
  model.shapes.clear();
  for (const auto& n : model.nodes) {
    switch (n.op) {
      case HG_OP_INPUT:
        ++inputs;
        require(n.inputs.empty(), "Input takes no inputs");
        require(!n.attrs.shape.empty(), "Input needs a shape attribute");
        model.shapes[n.id] = n.attrs.shape;
        break;
      case HG_OP_CONST_WEIGHT:
        require(!n.weight_ref.empty() && model.weights.count(n.weight_ref), "ConstWeight needs a resolvable weight_ref");
        model.shapes[n.id] = model.weights.at(n.weight_ref).dims;
        break;
      case HG_OP_ADD:
      case HG_OP_MULTIPLY: {
        require(n.inputs.size() == 2, "Add/Multiply take two inputs");
        auto a = model.shapes.at(n.inputs[0]);
        auto b = model.shapes.at(n.inputs[1]);
        require(a == b || elem_count(a) == 1 || elem_count(b) == 1,
                "shape mismatch at node " + n.id + ": " + shape_str(a) + " vs " + shape_str(b));
        model.shapes[n.id] = elem_count(a) == 1 ? b : a;
        break;
      }
      case HG_OP_SQUARE:
        require(n.inputs.size() == 1, "Square takes one input");
        model.shapes[n.id] = model.shapes.at(n.inputs[0]);
        break;
      case HG_OP_DOT: {
        require(n.inputs.size() == 1, "Dot takes one input");
        require(!n.weight_ref.empty() && model.weights.count(n.weight_ref), "Dot needs a resolvable weight_ref");
        const auto& w = model.weights.at(n.weight_ref);
        require(w.dims.size() == 2, "Dot weight must be (K,M)");
        auto in = model.shapes.at(n.inputs[0]);
        require(in.size() == 1 && in[0] == w.dims[0], "Dot inner dimension mismatch at node " + n.id);
        if (!n.bias_ref.empty()) {
          require(model.weights.count(n.bias_ref), "unresolvable bias_ref");
          require(elem_count(model.weights.at(n.bias_ref).dims) == w.dims[1], "bias shape mismatch at node " + n.id);
        }
        model.shapes[n.id] = {w.dims[1]};
        break;
      }
      case HG_OP_CONVOLUTION: {
        require(n.inputs.size() == 1, "Convolution takes one input");
        require(!n.weight_ref.empty() && model.weights.count(n.weight_ref),
                "Convolution needs a resolvable weight_ref");
        auto in = model.shapes.at(n.inputs[0]);
        const auto& w = model.weights.at(n.weight_ref);
        require(w.dims.size() == 4, "Convolution weight must be (F,C,KH,KW)");
        require(w.dims[0] == n.attrs.filters, "filter count mismatch");
        require(w.dims[1] == in[0], "channel count mismatch");
        require(w.dims[2] == n.attrs.window && w.dims[3] == n.attrs.window, "kernel window mismatch");
        if (!n.bias_ref.empty()) {
          require(model.weights.count(n.bias_ref), "unresolvable bias_ref");
          require(elem_count(model.weights.at(n.bias_ref).dims) == n.attrs.filters, "bias shape mismatch at node " + n.id);
        }
        require(in.size() == 3, "Convolution expects a (C,H,W) input");
        const u32 h = in[1] + n.attrs.pad[0] + n.attrs.pad[2];
        const u32 wd = in[2] + n.attrs.pad[1] + n.attrs.pad[3];
        require(n.attrs.window >= 1 && n.attrs.stride >= 1, "bad convolution attributes");
        require(h >= n.attrs.window && wd >= n.attrs.window, "window exceeds padded input");
        model.shapes[n.id] = {n.attrs.filters, (h - n.attrs.window) / n.attrs.stride + 1,
                              (wd - n.attrs.window) / n.attrs.stride + 1};
        break;
      }
      case HG_OP_RESHAPE: {
        require(n.inputs.size() == 1, "Reshape takes one input");
        require(elem_count(n.attrs.shape) == elem_count(model.shapes.at(n.inputs[0])),
                "Reshape changes the element count at node " + n.id);
        model.shapes[n.id] = n.attrs.shape;
        break;
      }
      case HG_OP_RELU:
        require(n.inputs.size() == 1, "Relu takes one input");
        model.shapes[n.id] = model.shapes.at(n.inputs[0]);
        break;
      case HG_OP_MAXPOOL: {
        require(n.inputs.size() == 1, "MaxPool takes one input");
        auto in = model.shapes.at(n.inputs[0]);
        require(in.size() == 3, "MaxPool expects a (C,H,W) input");
        const u32 stride = n.attrs.pool_stride ? n.attrs.pool_stride : n.attrs.window;
        require(n.attrs.window >= 1, "bad pooling window");
        require(in[1] >= n.attrs.window && in[2] >= n.attrs.window, "pooling window exceeds input");
        model.shapes[n.id] = {in[0], (in[1] - n.attrs.window) / stride + 1, (in[2] - n.attrs.window) / stride + 1};
        break;
      }
      case HG_OP_OUTPUT:
        ++outputs;
        require(n.inputs.size() == 1, "Output takes one input");
        model.shapes[n.id] = model.shapes.at(n.inputs[0]);
        break;
      default:
        throw Error(HG_ERR_VALIDATION, "unknown op");
    }
  }
  require(inputs == 1, "graph needs exactly one Input node");
  require(outputs == 1, "graph needs exactly one Output node");
  if (model.packing == HG_PACKING_COMPLEX) {
    for (const auto& n : model.nodes) {
      bool cc = n.op == HG_OP_SQUARE;
      if (n.op == HG_OP_MULTIPLY) {
        cc = model.node(n.inputs[0]).op != HG_OP_CONST_WEIGHT && model.node(n.inputs[1]).op != HG_OP_CONST_WEIGHT;
      }
      require(!cc, "complex packing cannot evaluate node " + n.id + " (cipher-cipher multiplication)");
    }
  }
  model.finalized = true;
}

// ---------------------------------------------------------------------------
// plan_rescaling (henet/graph.hpp:465-584)
// ---------------------------------------------------------------------------
static bool raises_scale(int op) {
  return op == HG_OP_SQUARE || op == HG_OP_DOT || op == HG_OP_CONVOLUTION || op == HG_OP_MULTIPLY;
}
static bool is_refresh(int op) { return op == HG_OP_RELU || op == HG_OP_MAXPOOL; }
static bool is_cipher_producing(const Model& m, const std::string& id) { return m.node(id).op != HG_OP_CONST_WEIGHT; }

static u64 elementary_products(const Model& m, const Node& n) {
  const auto& out = m.shapes.at(n.id);
  switch (n.op) {
    case HG_OP_SQUARE:
    case HG_OP_MULTIPLY:
      return elem_count(out);
    case HG_OP_DOT:
      return static_cast<u64>(m.shapes.at(n.inputs[0])[0]) * elem_count(out);
    case HG_OP_CONVOLUTION: {
      const auto& in = m.shapes.at(n.inputs[0]);
      u64 taps = 0;
      for (u32 y = 0; y < out[1]; ++y)
        for (u32 x = 0; x < out[2]; ++x)
          for (u32 ky = 0; ky < n.attrs.window; ++ky)
            for (u32 kx = 0; kx < n.attrs.window; ++kx) {
              const int64_t iy = static_cast<int64_t>(y * n.attrs.stride + ky) - n.attrs.pad[0];
              const int64_t ix = static_cast<int64_t>(x * n.attrs.stride + kx) - n.attrs.pad[1];
              if (iy >= 0 && iy < in[1] && ix >= 0 && ix < in[2]) ++taps;
            }
      return taps * in[0] * out[0];
    }
    default:
      return 0;
  }
}

static Plan plan_rescaling(const Context& ctx, const Model& model, int mode) {
  require(model.finalized, "model is not finalized");
  Plan plan;
  plan.mode = mode;
  const u32 top = static_cast<u32>(ctx.chain_len());
  std::map<std::string, bool> mult_downstream;
  for (auto it = model.nodes.rbegin(); it != model.nodes.rend(); ++it) mult_downstream[it->id] = false;
  for (auto it = model.nodes.rbegin(); it != model.nodes.rend(); ++it) {
    const Node& n = *it;
    for (const auto& in : n.inputs) {
      const bool contributes = raises_scale(n.op) || (!is_refresh(n.op) && mult_downstream[n.id]);
      if (contributes) mult_downstream[in] = true;
    }
  }
  const double s = ctx.default_scale;
  for (const auto& n : model.nodes) {
    NodePlan np;
    double scale_in = s;
    u32 level_in = top;
    bool first = true;
    for (const auto& in : n.inputs) {
      if (!is_cipher_producing(model, in)) continue;
      const auto& p = plan.nodes.at(in);
      if (first) {
        level_in = p.level_out;
        scale_in = p.scale_out;
        first = false;
      } else {
        require(p.level_out == level_in, "level mismatch between inputs of node " + n.id);
      }
    }
    np.level_in = level_in;
    np.level_out = level_in;
    np.scale_out = scale_in;
    if (is_refresh(n.op)) {
      np.level_out = top;
      np.scale_out = s;
    } else if (raises_scale(n.op)) {
      const bool cc = n.op == HG_OP_SQUARE || (n.op == HG_OP_MULTIPLY && is_cipher_producing(model, n.inputs[0]) &&
                                               is_cipher_producing(model, n.inputs[1]));
      const double raised = cc ? scale_in * scale_in : scale_in * s;
      const bool rescale_after = (mode == HG_RESCALE_NAIVE) || mult_downstream[n.id];
      np.decision = rescale_after ? HG_RESCALE_AFTER : HG_SKIP;
      if (rescale_after) {
        if (level_in < 2) throw Error(HG_ERR_VALIDATION, "infeasible depth: node " + n.id + " needs a rescale below level 1");
        np.level_out = level_in - 1;
        np.scale_out = raised / static_cast<double>(ctx.chain[level_in - 1]);
        plan.planned_rescale_ops += mode == HG_RESCALE_NAIVE ? elementary_products(model, n) : elem_count(model.shapes.at(n.id));
      } else {
        np.scale_out = raised;
      }
      if (static_cast<long double>(np.scale_out) >= ctx.modulus_products.at(np.level_out))
        throw Error(HG_ERR_VALIDATION, "infeasible depth: scale overflows q_level at node " + n.id);
    }
    plan.nodes[n.id] = np;
  }
  return plan;
}

// ---------------------------------------------------------------------------
// Executor (henet/graph.hpp:792-1117)
// ---------------------------------------------------------------------------
struct Value {
  bool is_cipher = false;
  CtBatch cipher;
  WeightTensor* plain = nullptr;
};

// (node id, ms) of the most recent hg_execute on this thread that asked for stats.
thread_local std::vector<std::pair<std::string, double>> g_last_layers;

// Batching of the Dot contraction over output positions (MacDenseTcArgs::npos and strides).
struct DotBatch {
  u32 npos = 1;
  u64 xk = 1, xp = 0, ym = 1, yp = 0;
  template <typename A>
  void apply(A& a) const {
    a.npos = npos;
    a.x_kstride = xk;
    a.x_pstride = xp;
    a.y_mstride = ym;
    a.y_pstride = yp;
  }
};

class Executor {
 public:
  Executor(const std::shared_ptr<Context>& ctx, Model& model, const Plan& plan, const RelinKeyDev* rk,
           hg_nonlin_fn provider, void* user, cudaStream_t s, bool timing)
      : ctx_(ctx), model_(model), plan_(plan), rk_(rk), provider_(provider), user_(user), s_(s), timing_(timing) {}

  CtBatch run(const CtBatch& input, hg_exec_stats* stats, std::array<double, 11>* node_ms) {
    require(model_.finalized, "model is not finalized");
    require(input.level == ctx_->chain_len(), "input must enter at the top level");
    require(input.packing == model_.packing, "input packing does not match the model");
    require(input.polys == 2, "input ciphertexts must have 2 polynomials");
    const Node* in_node = nullptr;
    for (const auto& n : model_.nodes)
      if (n.op == HG_OP_INPUT) in_node = &n;
    require(in_node != nullptr, "graph has no Input node");
    require(model_.shapes.at(in_node->id) == input.shape, "input shape does not match the model");
    const auto t0 = std::chrono::steady_clock::now();
    std::map<std::string, size_t> uses;
    for (const auto& n : model_.nodes)
      for (const auto& in : n.inputs) ++uses[in];

    // per-node CUDA events (ExecutionStats::layer_ms, henet/graph.hpp:860-866) when stats are
    // requested or HG_NODE_TIMING is set
    const bool timed = timing_ || stats != nullptr;
    std::vector<std::pair<const Node*, std::pair<cudaEvent_t, cudaEvent_t>>> evs;
    {
      std::lock_guard<std::mutex> g(*model_.mu);
      keep_ = model_.keep_encodings;
    }
    std::map<std::string, Value> values;
    u32 layer_seq = 0;
    const std::string out_id = [&] {
      for (const auto& n : model_.nodes)
        if (n.op == HG_OP_OUTPUT) return n.id;
      throw Error(HG_ERR_VALIDATION, "graph has no Output node");
    }();
    // HG_EXEC_TRACE=<ms>: host time per node of every execute that takes the host longer than <ms>
    static const double trace_ms = [] {
      const char* e = getenv("HG_EXEC_TRACE");
      return e ? atof(e) : -1.0;
    }();
    std::vector<std::pair<const Node*, double>> host_ms;
    for (const auto& n : model_.nodes) {
      const auto h0 = std::chrono::steady_clock::now();
      struct HostMark {
        std::vector<std::pair<const Node*, double>>* v;
        const Node* n;
        std::chrono::steady_clock::time_point t;
        ~HostMark() {
          if (v) v->emplace_back(n, std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count());
        }
      } host_mark{trace_ms >= 0 ? &host_ms : nullptr, &n, h0};
      cudaEvent_t e0 = nullptr, e1 = nullptr;
      if (timed) {
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, s_);
      }
      Value v;
      switch (n.op) {
        case HG_OP_INPUT:
          v.is_cipher = true;
          v.cipher = input;  // shares the caller's device buffer; never written
          v.cipher.shape = model_.shapes.at(n.id);
          break;
        case HG_OP_CONST_WEIGHT:
          v.plain = &model_.weights.at(n.weight_ref);
          break;
        case HG_OP_ADD:
        case HG_OP_MULTIPLY: {
          std::lock_guard<std::mutex> g(*model_.mu);  // lazily built weight state
          v = eval_elementwise(n, values);
          break;
        }
        case HG_OP_SQUARE:
          v = eval_square(n, values);
          break;
        case HG_OP_DOT:
        case HG_OP_CONVOLUTION: {
          std::lock_guard<std::mutex> g(*model_.mu);  // lazily built weight state
          v = eval_linear(n, values);
          break;
        }
        case HG_OP_RESHAPE:
        case HG_OP_OUTPUT:
          v = values.at(n.inputs[0]);
          v.cipher.shape = model_.shapes.at(n.id);
          break;
        case HG_OP_RELU:
        case HG_OP_MAXPOOL:
          v = eval_nonlinear(n, values, layer_seq++, stats);
          break;
        default:
          throw Error(HG_ERR_VALIDATION, "unknown op");
      }
      if (v.is_cipher) {
        require(v.cipher.level == plan_.nodes.at(n.id).level_out, "executed level diverged from the plan at node " + n.id);
      }
      if (timed) {
        cudaEventRecord(e1, s_);
        evs.push_back({&n, {e0, e1}});
      }
      for (const auto& in : n.inputs)
        if (--uses[in] == 0) values.erase(in);
      values[n.id] = std::move(v);
    }
    if (trace_ms >= 0) {
      double tot = 0;
      for (auto& h : host_ms) tot += h.second;
      if (tot > trace_ms) {
        std::string line = "[hg exec trace] host ms " + std::to_string(tot) + ":";
        for (auto& h : host_ms)
          if (h.second > 0.05) line += " " + h.first->id + "=" + std::to_string(h.second);
        fprintf(stderr, "%s\n", line.c_str());
      }
    }
    require(rescales_ == plan_.planned_rescale_ops, "executed rescale count diverged from the plan");
    auto it = values.find(out_id);
    require(it != values.end(), "output value missing");
    CtBatch out = std::move(it->second.cipher);
    values.clear();
    if (stats || timing_) {
      cuda_check(cudaStreamSynchronize(s_), "execute");
    }
    if (node_ms) node_ms->fill(0.0);
    g_last_layers.clear();
    for (auto& e : evs) {
      float ms = 0;
      cudaEventElapsedTime(&ms, e.second.first, e.second.second);
      if (node_ms) (*node_ms)[e.first->op] += ms;
      g_last_layers.emplace_back(e.first->id, static_cast<double>(ms));
      cudaEventDestroy(e.second.first);
      cudaEventDestroy(e.second.second);
    }
    if (stats) {
      stats->rescale_ops = rescales_;
      stats->relin_ops = relins_;
      stats->nonlin_elements += 0;
      stats->wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      stats->kernel_launches = launches_total() - launches0_;
    }
    return out;
  }

 private:
  // Dot / Convolution: mac_output over every output (henet/graph.hpp:905-993).
  // A weight tensor's device encoding for `key`, built by `build` -- per execute (the
  // reference's per-call WeightEncoder), or once per model and context when the model keeps
  // encodings (hg_model_keep_encodings; precompile_weights, henet/graph.hpp:657-679).
  BufPtr encoding(WeightTensor& w, std::vector<u64> key, size_t bytes, const std::function<void(void*)>& build) {
    key.insert(key.begin(), reinterpret_cast<u64>(ctx_.get()));
    if (!keep_) {
      BufPtr b = ctx_->alloc(bytes, s_);
      build(b->ptr);
      return b;
    }
    auto it = w.enc.find(key);
    if (it != w.enc.end()) {
      cuda_check(cudaStreamWaitEvent(s_, it->second.ready.get(), 0), "event");
      return it->second.buf;
    }
    // a kept encoding is allocated on the context's stream (it outlives any caller stream)
    KeptBuf k;
    k.buf = ctx_->alloc(bytes, ctx_->core->stream);
    if (s_ != ctx_->core->stream) cuda_check(cudaStreamWaitEvent(s_, record_ready(ctx_->core->stream).get(), 0), "event");
    build(k.buf->ptr);
    k.ready = record_ready(s_);
    w.enc[key] = k;
    return k.buf;
  }
  static u64 bits(double d) {
    u64 u;
    std::memcpy(&u, &d, 8);
    return u;
  }

  Value eval_linear(const Node& n, std::map<std::string, Value>& values) {
    const Context& ctx = *ctx_;
    const CtBatch& x = values.at(n.inputs[0]).cipher;
    const auto& np = plan_.nodes.at(n.id);
    const bool naive = plan_.mode == HG_RESCALE_NAIVE;
    const bool layer_rescale = np.decision == HG_RESCALE_AFTER;
    WeightTensor& w = model_.weights.at(n.weight_ref);
    WeightTensor* b = n.bias_ref.empty() ? nullptr : &model_.weights.at(n.bias_ref);
    if (naive && layer_rescale) return eval_linear_naive(n, x, w, b);
    const double s = ctx.default_scale;
    const u32 L = x.level;
    const u32 N = ctx.n;
    const auto& out_shape = model_.shapes.at(n.id);
    const u64 M = elem_count(out_shape);

    check_scalar_encodable(ctx, w.max_abs, L, s);
    const double acc_scale = x.scale * s;  // term.scale = x.scale * pt.scale (henet/ckks.hpp:384)

    Value v;
    v.is_cipher = true;
    v.cipher.packing = x.packing;
    v.cipher.scale = acc_scale;
    v.cipher.shape = out_shape;
    ensure(ctx, v.cipher, M, 2, L, s_);

    const float* wd = weight_dev(ctx, w, s_);
    BufPtr bias_res;
    BufPtr bias_pt;

    const size_t wb = ctx.word_bytes();
    // The Dot contraction (henet/graph.hpp:935-954) of x with weight residues wres [L][K][Mpad]
    // and bias_res [L][Mpad] into v.  bt batches it over output positions (a 1x1, stride-1
    // convolution: one Dot per position, positions as extra columns of the same kernels);
    // tag keeps the packed-weight cache keys of the two uses apart.
    auto dot_dispatch = [&](WeightTensor& w, const BufPtr& wres, const BufPtr& bias_res, u32 K, u32 Mo, u32 Mpad,
                            u64 tag, const DotBatch& bt) -> int {
      int r = 1;
      if (ctx.wide) {
        // Limbs whose prime is < 2^30 (BASELINE c4/c5b: limbs 1..7) go through the int8 tensor
        // cores on a u32 copy of their residues; the rest (the 40-bit limb 0) on the wide
        // CUDA-core kernel.
        u32 tc_lo = L;
        if (ctx.dense_tc && K <= 8192 && L >= 2) {
          tc_lo = 1;
          for (u32 i = 1; i < L; ++i)
            if (ctx.chain[i] >= (1ull << 30)) tc_lo = L;
          if (ctx.chain[0] < (1ull << 30)) tc_lo = L;  // all narrow: no wide context would exist
        }
        MacDenseArgsW a{};
        a.X = x.data64();
        a.Y = v.cipher.data64();
        a.W = static_cast<const u64*>(wres->ptr);
        a.bias = bias_res ? static_cast<const u64*>(bias_res->ptr) : nullptr;
        a.K = K;
        a.M = Mo;
        a.Mpad = Mpad;
        a.N = N;
        a.level = L;
        a.polys = 2;
        a.x_level = x.level;
        a.limb_lo = 0;
        a.limb_cnt = tc_lo;
        for (u32 i = 0; i < L; ++i) {  // 128-bit sums of K products (< (q-1)^2 each)
          const long double qm1 = static_cast<long double>(ctx.chain[i] - 1);
          a.fold[i] = (qm1 * qm1 * K + ctx.chain[i] >= 0x1p128L) ? 1 : 0;
        }
        // the 40-bit limb itself on the tensor cores (5 byte planes, k_mac_dense_tc_w) when
        // the rest of the layer is there too and K keeps its diagonal sums < 2^31
        static const bool wide_tc = [] {
          const char* e = getenv("HG_WIDE_TC");
          return !(e != nullptr && e[0] == '0');
        }();
        const bool limb0_tc = wide_tc && tc_lo == 1 && ctx.chain[0] < (1ull << 40) && K <= 6605;
        if (bt.npos > 1 && !limb0_tc) return -2;  // the CUDA-core wide kernels run plain Dots only
        if (limb0_tc) {
          BufPtr wp0 = ctx.alloc(tc_packed_weight_bytes_w(K, Mo), s_);
          check_launch(launch_pack_weights_tc_w(static_cast<const u64*>(wres->ptr), static_cast<uint8_t*>(wp0->ptr), K,
                                                Mo, Mpad, s_),
                       "pack weights (wide)");
          MacDenseTcWArgs t{};
          t.X = x.data64();
          t.Y = v.cipher.data64();
          t.Wp = static_cast<const uint8_t*>(wp0->ptr);
          t.bias = bias_res ? static_cast<const u64*>(bias_res->ptr) : nullptr;  // limb 0 row
          t.K = K;
          t.M = Mo;
          t.Mpad = Mpad;
          t.N = N;
          t.level = L;
          t.polys = 2;
          t.x_level = x.level;
          t.limb = 0;
          const u64 q0 = ctx.chain[0];
          u64 c = 1;
          for (int i = 0; i < 9; ++i) {
            t.cs[i] = c;
            c = static_cast<u64>((static_cast<nt::u128>(c) << 8) % q0);
          }
          bt.apply(t);
          r = launch_mac_dense_tc_w(t, &ctx.basisw.p[0], s_);
        } else {
          r = launch_mac_dense_w(a, ctx.basisw, s_);
        }
        if (r >= 0 && tc_lo < L) {
          check_launch(r, "mac_dense_w");
          const u32 cnt = L - tc_lo;
          // the kernel reads and writes those limbs of the u64 tensors in place; u32 copies
          // of the (small) weights [cnt][K][Mpad] and bias [cnt][Mpad]
          BufPtr wn = ctx.alloc(static_cast<u64>(cnt) * K * Mpad * 4, s_);
          check_launch(launch_limbs_to_u32(static_cast<const u64*>(wres->ptr), static_cast<u32*>(wn->ptr), 1, L, tc_lo,
                                           cnt, static_cast<u32>(static_cast<u64>(K) * Mpad), s_),
                       "narrow weights");
          BufPtr bn;
          if (bias_res) {
            bn = ctx.alloc(static_cast<u64>(cnt) * Mpad * 4, s_);
            check_launch(launch_limbs_to_u32(static_cast<const u64*>(bias_res->ptr), static_cast<u32*>(bn->ptr), 1, L,
                                             tc_lo, cnt, Mpad, s_),
                         "narrow bias");
          }
          BufPtr wp = ctx.alloc(tc_packed_weight_bytes(K, Mo, cnt), s_);
          check_launch(launch_pack_weights_tc(static_cast<const u32*>(wn->ptr), static_cast<uint8_t*>(wp->ptr), K, Mo,
                                              Mpad, cnt, s_),
                       "pack weights");
          Basis sub{};  // the narrow constants of limbs tc_lo.. (every basis entry < 2^32 is valid)
          for (u32 i = 0; i < cnt; ++i) sub.p[i] = ctx.basis.p[tc_lo + i];
          MacDenseTcArgs t{};
          t.X64 = x.data64();
          t.Y64 = v.cipher.data64();
          t.limb_off = tc_lo;
          t.y_level = L;
          t.Wp = static_cast<const uint8_t*>(wp->ptr);
          t.bias = bn ? static_cast<const u32*>(bn->ptr) : nullptr;
          t.K = K;
          t.M = Mo;
          t.Mpad = Mpad;
          t.N = N;
          t.level = cnt;
          t.polys = 2;
          t.x_level = x.level;
          for (u32 i = 0; i < cnt; ++i) t.planes[i] = ctx.chain[tc_lo + i] < (1ull << 24) ? 3 : 4;
          bt.apply(t);
          r = launch_mac_dense_tc(t, sub, s_);
        }
      } else if (ctx.dense_tc && K <= 8192) {
        // tensor-core path: byte-plane weights packed once per call, then tcgen05.mma.kind::i8
        BufPtr wp = encoding(w, {tag + 3, L, bits(s), Mpad}, tc_packed_weight_bytes(K, Mo, L), [&](void* p) {
          check_launch(launch_pack_weights_tc(static_cast<const u32*>(wres->ptr), static_cast<uint8_t*>(p), K, Mo,
                                              Mpad, L, s_),
                       "pack weights");
        });
        MacDenseTcArgs a{};
        a.X = x.data();
        a.Y = v.cipher.data();
        a.Wp = static_cast<const uint8_t*>(wp->ptr);
        a.bias = bias_res ? static_cast<const u32*>(bias_res->ptr) : nullptr;
        a.K = K;
        a.M = Mo;
        a.Mpad = Mpad;
        a.N = N;
        a.level = L;
        a.polys = 2;
        a.x_level = x.level;
        for (u32 i = 0; i < L; ++i) a.planes[i] = ctx.chain[i] < (1ull << 24) ? 3 : 4;
        bt.apply(a);
        r = launch_mac_dense_tc(a, ctx.basis, s_);
      } else {
        if (bt.npos > 1) return -2;  // the CUDA-core kernel runs plain Dots only
        MacDenseArgs a{};
        a.X = x.data();
        a.Y = v.cipher.data();
        a.W = static_cast<const u32*>(wres->ptr);
        a.bias = bias_res ? static_cast<const u32*>(bias_res->ptr) : nullptr;
        a.K = K;
        a.M = Mo;
        a.Mpad = Mpad;
        a.N = N;
        a.level = L;
        a.polys = 2;
        a.x_level = x.level;
        for (u32 i = 0; i < L; ++i) {
          const long double qm1 = static_cast<long double>(ctx.chain[i] - 1);
          a.fold[i] = (qm1 * qm1 * K >= 18446744073709551616.0L) ? 1 : 0;
        }
        r = launch_mac_dense(a, ctx.basis, s_);
      }
      return r;
    };

    if (n.op == HG_OP_DOT) {
      const u32 K = w.dims[0], Mo = w.dims[1];
      const u32 BM = ctx.wide ? mac_dense_w_bm() : mac_dense_warps(Mo) * 4;
      const u32 Mpad = (Mo + BM - 1) / BM * BM;
      BufPtr wres = encoding(w, {1, L, bits(s), Mpad}, static_cast<u64>(L) * K * Mpad * wb, [&](void* p) {
        cuda_check(cudaMemsetAsync(p, 0, static_cast<u64>(L) * K * Mpad * wb, s_), "memset");
        check_launch(encode_f32(ctx, wd, w.data.size(), Mo, Mpad, static_cast<u64>(K) * Mpad, L, s, p, s_),
                     "encode weights");
      });
      int r = 1;
      if (b && x.packing == HG_PACKING_REAL) {
        check_scalar_encodable(ctx, b->max_abs, L, acc_scale);
        const float* bd = weight_dev(ctx, *b, s_);
        bias_res = encoding(*b, {2, L, bits(acc_scale), Mpad}, static_cast<u64>(L) * Mpad * wb, [&](void* p) {
          check_launch(encode_f32(ctx, bd, Mo, Mo, Mpad, Mpad, L, acc_scale, p, s_), "encode bias");
        });
      }
      r = dot_dispatch(w, wres, bias_res, K, Mo, Mpad, 0, DotBatch{});
      check_launch(r, "mac_dense");
    } else {
      const auto& in_shape = x.shape;
      require(in_shape.size() == 3, "Convolution expects a (C,H,W) input");
      const u32 F = n.attrs.filters, C = in_shape[0], win = n.attrs.window, T2 = win * win;
      // 1x1, stride-1, unpadded windows (the MobileNetV2 expand / project layers): every output
      // position is a Dot of its C input channels, so the layer runs as one batched Dot on the
      // tensor-core contraction (positions as extra columns) instead of the tap-gather kernel.
      bool conv1x1_done = false;
      static const bool conv1x1_on = [] {
        const char* e = getenv("HG_CONV1X1_DOT");
        return !(e != nullptr && e[0] == '0');
      }();
      if (conv1x1_on && win == 1 && n.attrs.stride == 1 && n.attrs.pad[0] == 0 && n.attrs.pad[1] == 0 &&
          n.attrs.pad[2] == 0 && n.attrs.pad[3] == 0 && in_shape[1] == out_shape[1] && in_shape[2] == out_shape[2]) {
        const u32 K = C, Mo = F;
        const u32 BM = ctx.wide ? mac_dense_w_bm() : mac_dense_warps(Mo) * 4;
        const u32 Mpad = (Mo + BM - 1) / BM * BM;
        // weights [F][C] -> [C][F] (the Dot layout [K][M]), then encoded like a Dot's
        BufPtr wt = encoding(w, {109}, static_cast<u64>(K) * Mo * 4, [&](void* p) {
          std::vector<float> t(static_cast<u64>(K) * Mo);
          for (u32 f = 0; f < F; ++f)
            for (u32 c = 0; c < C; ++c) t[static_cast<u64>(c) * F + f] = w.data[static_cast<u64>(f) * C + c];
          cuda_check(cudaMemcpyAsync(p, t.data(), t.size() * 4, cudaMemcpyHostToDevice, s_), "h2d");
          cuda_check(cudaStreamSynchronize(s_), "h2d");  // the host vector leaves scope
        });
        BufPtr wres = encoding(w, {101, L, bits(s), Mpad}, static_cast<u64>(L) * K * Mpad * wb, [&](void* p) {
          cuda_check(cudaMemsetAsync(p, 0, static_cast<u64>(L) * K * Mpad * wb, s_), "memset");
          check_launch(encode_f32(ctx, static_cast<const float*>(wt->ptr), static_cast<u64>(K) * Mo, Mo, Mpad,
                                  static_cast<u64>(K) * Mpad, L, s, p, s_),
                       "encode weights");
        });
        BufPtr bres;
        if (b && x.packing == HG_PACKING_REAL) {
          check_scalar_encodable(ctx, b->max_abs, L, acc_scale);
          const float* bd = weight_dev(ctx, *b, s_);
          bres = encoding(*b, {102, L, bits(acc_scale), Mpad}, static_cast<u64>(L) * Mpad * wb, [&](void* p) {
            check_launch(encode_f32(ctx, bd, Mo, Mo, Mpad, Mpad, L, acc_scale, p, s_), "encode bias");
          });
        }
        const u32 HW = in_shape[1] * in_shape[2];
        DotBatch bt;
        bt.npos = HW;
        bt.xk = HW;  // input channel c of position p: element c * HW + p
        bt.xp = 1;
        bt.ym = HW;  // output filter f of position p: element f * HW + p
        bt.yp = 1;
        const int r = dot_dispatch(w, wres, bres, K, Mo, Mpad, 100, bt);
        if (r != -2) {
          check_launch(r, "mac_conv1x1");
          conv1x1_done = true;
        }
      }
      if (!conv1x1_done) {
      // one launch of the convolution kernel on (X, Y, Wr, Bi) with Cc channels, Ff filters
      auto run_conv = [&](const void* X, void* Y, const void* Wr, const void* Bi, u32 Cc, u32 Ff, u32 groups = 1,
                          u64 gx = 0, u64 gy = 0, u64 gw = 0, u64 gb = 0) {
        int r = 1;
        if (ctx.wide) {
          MacConvArgsW a{};
          a.groups = groups;
          a.gx = gx;
          a.gy = gy;
          a.gw = gw;
          a.gb = gb;
          a.X = static_cast<const u64*>(X);
          a.Y = static_cast<u64*>(Y);
          a.W = static_cast<const u64*>(Wr);
          a.bias = static_cast<const u64*>(Bi);
          a.C = Cc;
          a.IH = in_shape[1];
          a.IW = in_shape[2];
          a.F = Ff;
          a.OH = out_shape[1];
          a.OW = out_shape[2];
          a.win = win;
          a.stride = n.attrs.stride;
          a.pad_top = n.attrs.pad[0];
          a.pad_left = n.attrs.pad[1];
          a.level = L;
          a.polys = 2;
          a.x_level = x.level;
          a.N = N;
          for (u32 i = 0; i < L; ++i) {
            const long double qm1 = static_cast<long double>(ctx.chain[i] - 1);
            a.fold[i] = (qm1 * qm1 * (static_cast<long double>(Cc) * T2) + ctx.chain[i] >= 0x1p128L) ? 1 : 0;
          }
          r = launch_mac_conv_w(a, ctx.basisw, s_);
        } else {
          MacConvArgs a{};
          a.X = static_cast<const u32*>(X);
          a.Y = static_cast<u32*>(Y);
          a.W = static_cast<const u32*>(Wr);
          a.bias = static_cast<const u32*>(Bi);
          a.C = Cc;
          a.IH = in_shape[1];
          a.IW = in_shape[2];
          a.F = Ff;
          a.OH = out_shape[1];
          a.OW = out_shape[2];
          a.win = win;
          a.stride = n.attrs.stride;
          a.pad_top = n.attrs.pad[0];
          a.pad_left = n.attrs.pad[1];
          a.level = L;
          a.polys = 2;
          a.x_level = x.level;
          a.N = N;
          // valid-tap table per output position (geometry only; henet/graph.hpp:976-989),
          // cached on the context: (input element, window tap), ascending per position
          {
            const u32 npos = a.OH * a.OW;
            // entries carry the input's word offset (element * polys * x_level * N): no address
            // multiply per tap in the kernel
            const u64 xstride = static_cast<u64>(a.polys) * a.x_level * a.N;
            require(static_cast<u64>(Cc) * a.IH * a.IW * xstride < (1ull << 32),
                    "convolution input too large for 32-bit tap offsets");
            const std::vector<u32> key = {Cc, a.IH, a.IW, a.OH, a.OW, win, a.stride, a.pad_top, a.pad_left,
                                          static_cast<u32>(xstride)};
            std::lock_guard<std::mutex> g(ctx.geo_mu);
            BufPtr& tb = ctx.geo_cache[key];
            const size_t toff = ((npos + 1) * 4 + 15) / 16 * 16;
            if (!tb) {
              std::vector<u32> tab(npos + 1);
              std::vector<uint2> taps;
              for (u32 oy = 0; oy < a.OH; ++oy)
                for (u32 ox = 0; ox < a.OW; ++ox) {
                  for (u32 c = 0; c < Cc; ++c)
                    for (u32 ky = 0; ky < win; ++ky)
                      for (u32 kx = 0; kx < win; ++kx) {
                        const int iy = static_cast<int>(oy * a.stride + ky) - static_cast<int>(a.pad_top);
                        const int ix = static_cast<int>(ox * a.stride + kx) - static_cast<int>(a.pad_left);
                        if (iy < 0 || iy >= static_cast<int>(a.IH) || ix < 0 || ix >= static_cast<int>(a.IW)) continue;
                        taps.push_back(make_uint2(
                            static_cast<u32>(((c * a.IH + static_cast<u32>(iy)) * a.IW + static_cast<u32>(ix)) * xstride),
                            (c * win + ky) * win + kx));
                      }
                  tab[oy * a.OW + ox + 1] = static_cast<u32>(taps.size());
                }
              tb = ctx.alloc(toff + taps.size() * 8 + 16, s_);
              cuda_check(cudaMemcpyAsync(tb->ptr, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice, s_), "taps");
              if (!taps.empty())
                cuda_check(cudaMemcpyAsync(static_cast<char*>(tb->ptr) + toff, taps.data(), taps.size() * 8,
                                           cudaMemcpyHostToDevice, s_),
                           "taps");
              cuda_check(cudaStreamSynchronize(s_), "taps");  // host vectors leave scope
            }
            a.tap_off = static_cast<const u32*>(tb->ptr);
            a.taps = reinterpret_cast<const uint2*>(static_cast<const char*>(tb->ptr) + toff);
          }
          static const bool fp64_on = [] {
            const char* e = getenv("HG_CONV_FP64");
            return !(e != nullptr && e[0] == '0');
          }();
          for (u32 i = 0; i < L; ++i) {
            const long double qm1 = static_cast<long double>(ctx.chain[i] - 1);
            const u32 taps = Cc * win * win;
            a.fold[i] = (qm1 * qm1 * taps >= 18446744073709551616.0L) ? 1 : 0;
            // a sum of `taps` products of residues is an integer < 2^53: exact in double
            a.fp64[i] = (fp64_on && taps <= 32 && qm1 * qm1 * taps < 9007199254740992.0L) ? 1 : 0;
          }
          r = launch_mac_conv(a, ctx.basis, s_);
        }
        check_launch(r, "mac_conv");
      };
      // Depthwise weights (F == C, w[f][c] == 0 for f != c): the reference evaluates them as a
      // full convolution whose off-diagonal taps are exact zeros (it has no grouped
      // convolution); a zero residue adds nothing to a canonical sum, so each
      // channel runs as its own 1 -> 1 convolution on its slices (9 taps instead of 9 C).
      if (w.depthwise < 0) {
        bool dw = F == C && C > 1;
        for (u32 f = 0; dw && f < F; ++f)
          for (u32 c = 0; dw && c < C; ++c)
            if (c != f)
              for (u32 t = 0; dw && t < T2; ++t) dw = w.data[(static_cast<u64>(f) * C + c) * T2 + t] == 0.0f;
        w.depthwise = dw ? 1 : 0;
      }
      if (w.depthwise == 1) {
        BufPtr dg = encoding(w, {6}, static_cast<u64>(C) * T2 * 4, [&](void* p) {
          std::vector<float> diag(static_cast<u64>(C) * T2);
          for (u32 c = 0; c < C; ++c)
            for (u32 t = 0; t < T2; ++t) diag[c * T2 + t] = w.data[(static_cast<u64>(c) * C + c) * T2 + t];
          cuda_check(cudaMemcpyAsync(p, diag.data(), diag.size() * 4, cudaMemcpyHostToDevice, s_), "h2d");
          cuda_check(cudaStreamSynchronize(s_), "h2d");  // the host vector leaves scope
        });
        // residues per channel: [C][L][T2] (a channel's slice is a [L][T2] weight table)
        BufPtr wres = encoding(w, {7, L, bits(s)}, static_cast<u64>(C) * L * T2 * wb, [&](void* p) {
          check_launch(encode_f32(ctx, static_cast<const float*>(dg->ptr), static_cast<u64>(C) * T2, T2, L * T2, T2, L,
                                  s, p, s_),
                       "encode weights");
        });
        if (b && x.packing == HG_PACKING_REAL) {
          check_scalar_encodable(ctx, b->max_abs, L, acc_scale);
          const float* bd = weight_dev(ctx, *b, s_);
          bias_res = encoding(*b, {8, L, bits(acc_scale)}, static_cast<u64>(C) * L * wb, [&](void* p) {
            check_launch(encode_f32(ctx, bd, C, 1, L, 1, L, acc_scale, p, s_), "encode bias");  // [C][L]
          });
        }
        const u64 xs = static_cast<u64>(in_shape[1]) * in_shape[2] * 2 * x.level * N * wb;  // bytes per channel
        const u64 ys = static_cast<u64>(out_shape[1]) * out_shape[2] * 2 * L * N * wb;
        if (ctx.wide) {
          // every channel in one launch (groups = C): 96 launches of one channel's positions
          // each left the GPU mostly idle
          run_conv(x.buf->ptr, v.cipher.buf->ptr, wres->ptr, bias_res ? bias_res->ptr : nullptr, 1, 1, C, xs / wb,
                   ys / wb, static_cast<u64>(L) * T2, L);
        } else {
          for (u32 c = 0; c < C; ++c)
            run_conv(static_cast<const char*>(x.buf->ptr) + c * xs, static_cast<char*>(v.cipher.buf->ptr) + c * ys,
                     static_cast<const char*>(wres->ptr) + static_cast<u64>(c) * L * T2 * wb,
                     bias_res ? static_cast<const char*>(bias_res->ptr) + static_cast<u64>(c) * L * wb : nullptr, 1, 1);
        }
      } else {
        BufPtr wres = encoding(w, {4, L, bits(s)}, static_cast<u64>(L) * w.data.size() * wb, [&](void* p) {
          check_launch(encode_f32(ctx, wd, w.data.size(), static_cast<u32>(w.data.size()),
                                  static_cast<u32>(w.data.size()), w.data.size(), L, s, p, s_),
                       "encode weights");
        });
        if (b && x.packing == HG_PACKING_REAL) {
          check_scalar_encodable(ctx, b->max_abs, L, acc_scale);
          const float* bd = weight_dev(ctx, *b, s_);
          bias_res = encoding(*b, {5, L, bits(acc_scale)}, static_cast<u64>(L) * F * wb, [&](void* p) {
            check_launch(encode_f32(ctx, bd, F, F, F, F, L, acc_scale, p, s_), "encode bias");
          });
        }
        run_conv(x.buf->ptr, v.cipher.buf->ptr, wres->ptr, bias_res ? bias_res->ptr : nullptr, C, F);
      }
      }  // !conv1x1_done
    }
    if (b && x.packing == HG_PACKING_COMPLEX) {
      // encode_broadcast under complex packing: encode_vector of (b + b i) in every slot
      // (henet/encoding.hpp:275-283) at (level, acc.scale); one plaintext per bias value.
      const u64 nb = b->data.size();
      std::vector<double> slots(nb * ctx.n);
      for (u64 i = 0; i < nb; ++i)
        for (u32 j = 0; j < ctx.n / 2; ++j) {
          slots[(i * ctx.n / 2 + j) * 2] = b->data[i];
          slots[(i * ctx.n / 2 + j) * 2 + 1] = b->data[i];
        }
      BufPtr ds = ctx.alloc(slots.size() * sizeof(double), s_);
      cuda_check(cudaMemcpyAsync(ds->ptr, slots.data(), slots.size() * sizeof(double), cudaMemcpyHostToDevice, s_),
                 "h2d");
      std::vector<unsigned long long> mant;
      std::vector<int> ex;
      bias_pt = encode_vectors_dev(ctx, static_cast<const double*>(ds->ptr), ctx.n / 2, nb, L, acc_scale, s_, mant, ex);
      EwArgs e{};
      e.op = EwOp::AddVector;
      e.a = v.cipher.data();
      e.b = static_cast<const u32*>(bias_pt->ptr);
      e.per_element = 1;
      e.pt_div = n.op == HG_OP_DOT ? 1 : out_shape[1] * out_shape[2];
      e.out = v.cipher.data();
      e.count = M;
      e.polys_a = 2;
      e.polys_out = 2;
      e.level = L;
      run_ew(ctx, e, s_);
    }
    if (layer_rescale) {
      v.cipher = do_rescale(ctx, v.cipher, L - 1, s_);
      rescales_ += M;
    }
    return v;
  }

  // Naive plan (mac_output, henet/graph.hpp:905-933, naive && RescaleAfter): every product
  // x[i] * enc(w) is rescaled before it is accumulated; the bias goes in afterwards at the
  // rescaled level and scale.  Round r multiplies every output's r-th tap (ascending
  // eval_dot / eval_convolution order; a zero term where an output has fewer taps, and
  // rescale(0) = 0), rescales the M terms as one batch and adds them into the accumulators.
  Value eval_linear_naive(const Node& n, const CtBatch& x, WeightTensor& w, WeightTensor* b) {
    const Context& ctx = *ctx_;
    require(x.level >= 2, "cannot rescale below level 1");
    const size_t wb = ctx.word_bytes();
    const double s = ctx.default_scale;
    const u32 L = x.level;
    const auto& out_shape = model_.shapes.at(n.id);
    const u64 M = elem_count(out_shape);
    check_scalar_encodable(ctx, w.max_abs, L, s);
    std::vector<std::vector<std::pair<u32, u32>>> taps(M);  // (input element, weight index)
    if (n.op == HG_OP_DOT) {
      const u32 K = w.dims[0], Mo = w.dims[1];
      for (u32 m = 0; m < Mo; ++m)
        for (u32 k = 0; k < K; ++k) taps[m].emplace_back(k, k * Mo + m);
    } else {
      const auto& in = x.shape;
      require(in.size() == 3, "Convolution expects a (C,H,W) input");
      const u32 F = n.attrs.filters, C = in[0], IH = in[1], IW = in[2], win = n.attrs.window;
      const u32 OH = out_shape[1], OW = out_shape[2];
      for (u32 f = 0; f < F; ++f)
        for (u32 oy = 0; oy < OH; ++oy)
          for (u32 ox = 0; ox < OW; ++ox)
            for (u32 c = 0; c < C; ++c)
              for (u32 ky = 0; ky < win; ++ky)
                for (u32 kx = 0; kx < win; ++kx) {
                  const int iy = static_cast<int>(oy * n.attrs.stride + ky) - static_cast<int>(n.attrs.pad[0]);
                  const int ix = static_cast<int>(ox * n.attrs.stride + kx) - static_cast<int>(n.attrs.pad[1]);
                  if (iy < 0 || iy >= static_cast<int>(IH) || ix < 0 || ix >= static_cast<int>(IW)) continue;
                  taps[(f * OH + oy) * OW + ox].emplace_back((c * IH + static_cast<u32>(iy)) * IW + static_cast<u32>(ix),
                                                             ((f * C + c) * win + ky) * win + kx);
                }
    }
    u64 R = 0, terms = 0;
    for (const auto& t : taps) {
      require(!t.empty(), "empty accumulation");
      R = std::max<u64>(R, t.size());
      terms += t.size();
    }
    std::vector<u32> gidx(R * M, 0xFFFFFFFFu), gw(R * M, 0u);
    for (u64 m = 0; m < M; ++m)
      for (u64 r = 0; r < taps[m].size(); ++r) {
        gidx[r * M + m] = taps[m][r].first;
        gw[r * M + m] = taps[m][r].second;
      }
    BufPtr tab = ctx.alloc(2 * R * M * 4, s_);
    u32* d_gidx = static_cast<u32*>(tab->ptr);
    u32* d_gw = d_gidx + R * M;
    cuda_check(cudaMemcpyAsync(d_gidx, gidx.data(), R * M * 4, cudaMemcpyHostToDevice, s_), "h2d");
    cuda_check(cudaMemcpyAsync(d_gw, gw.data(), R * M * 4, cudaMemcpyHostToDevice, s_), "h2d");
    // weight residues element-major [count][L]
    const float* wd = weight_dev(ctx, w, s_);
    const u64 wc = w.data.size();
    BufPtr wres = ctx.alloc(wc * L * wb, s_);
    check_launch(encode_f32(ctx, wd, wc, 1, L, 1, L, s, wres->ptr, s_), "encode weights");

    CtBatch term;
    term.packing = x.packing;
    term.scale = x.scale * s;  // term.scale = x.scale * pt.scale (henet/ckks.hpp:384)
    ensure(ctx, term, M, 2, L, s_);
    CtBatch acc;
    for (u64 r = 0; r < R; ++r) {
      EwArgs e{};
      e.op = EwOp::GatherMul;
      e.a = x.data();
      e.res = static_cast<const u32*>(wres->ptr);
      e.gidx = d_gidx + r * M;
      e.gw = d_gw + r * M;
      e.out = term.data();
      e.count = M;
      e.polys_a = 2;
      e.polys_out = 2;
      e.level = L;
      run_ew(ctx, e, s_);
      CtBatch t = do_rescale(ctx, term, L - 1, s_);
      if (r == 0) {
        acc = t;
      } else {
        EwArgs a{};
        a.op = EwOp::AddCC;
        a.a = acc.data();
        a.b = t.data();
        a.out = acc.data();
        a.count = M;
        a.polys_a = 2;
        a.polys_out = 2;
        a.level = L - 1;
        run_ew(ctx, a, s_);
      }
    }
    rescales_ += terms;
    acc.shape = out_shape;
    acc.packing = x.packing;
    if (b) {
      const u32 bl = L - 1;
      check_scalar_encodable(ctx, b->max_abs, bl, acc.scale);
      const u32 pt_div = n.op == HG_OP_DOT ? 1 : out_shape[1] * out_shape[2];
      EwArgs e{};
      e.a = acc.data();
      e.out = acc.data();
      e.per_element = 1;
      e.pt_div = pt_div;
      e.count = M;
      e.polys_a = 2;
      e.polys_out = 2;
      e.level = bl;
      BufPtr bias_res;
      if (x.packing == HG_PACKING_REAL) {
        // encode_broadcast of a real scalar: the expanded constant (henet/encoding.hpp:210-219)
        const float* bd = weight_dev(ctx, *b, s_);
        bias_res = ctx.alloc(b->data.size() * bl * wb, s_);
        check_launch(encode_f32(ctx, bd, b->data.size(), 1, bl, 1, bl, acc.scale, bias_res->ptr, s_), "encode bias");
        e.op = EwOp::AddScalar;
        e.res = static_cast<const u32*>(bias_res->ptr);
      } else {
        bias_res = complex_bias(*b, bl, acc.scale);
        e.op = EwOp::AddVector;
        e.b = static_cast<const u32*>(bias_res->ptr);
      }
      run_ew(ctx, e, s_);
      cuda_check(cudaStreamSynchronize(s_), "bias");  // host-side bias buffers leave scope
    }
    Value v;
    v.is_cipher = true;
    v.cipher = acc;
    return v;
  }

  // encode_broadcast under complex packing: encode_vector of (b + b i) in every slot
  // (henet/encoding.hpp:275-283) at (level, scale); one plaintext per bias value.
  BufPtr complex_bias(const WeightTensor& b, u32 level, double scale) {
    const Context& ctx = *ctx_;
    const u64 nb = b.data.size();
    std::vector<double> slots(nb * ctx.n);
    for (u64 i = 0; i < nb; ++i)
      for (u32 j = 0; j < ctx.n / 2; ++j) {
        slots[(i * ctx.n / 2 + j) * 2] = b.data[i];
        slots[(i * ctx.n / 2 + j) * 2 + 1] = b.data[i];
      }
    BufPtr ds = ctx.alloc(slots.size() * sizeof(double), s_);
    cuda_check(cudaMemcpyAsync(ds->ptr, slots.data(), slots.size() * sizeof(double), cudaMemcpyHostToDevice, s_),
               "h2d");
    std::vector<unsigned long long> mant;
    std::vector<int> ex;
    BufPtr pt = encode_vectors_dev(ctx, static_cast<const double*>(ds->ptr), ctx.n / 2, nb, level, scale, s_, mant, ex);
    cuda_check(cudaStreamSynchronize(s_), "bias");  // the host slot vector leaves scope
    return pt;
  }

  Value eval_square(const Node& n, std::map<std::string, Value>& values) {
    const CtBatch& x = values.at(n.inputs[0]).cipher;
    const auto& np = plan_.nodes.at(n.id);
    require(rk_ != nullptr, "graph contains cipher-cipher products but no relin key");
    check_cc_mul(x);
    Value v;
    v.is_cipher = true;
    const bool rs = np.decision == HG_RESCALE_AFTER;
    v.cipher = do_relin(*ctx_, *rk_, &x, &x, 1, rs, s_);
    v.cipher.shape = x.shape;
    relins_ += x.count;
    if (rs) rescales_ += x.count;
    return v;
  }

  Value eval_elementwise(const Node& n, std::map<std::string, Value>& values) {
    const Context& ctx = *ctx_;
    const Value& a = values.at(n.inputs[0]);
    const Value& b = values.at(n.inputs[1]);
    require(a.is_cipher || b.is_cipher, "constant-only op " + n.id);
    const auto& np = plan_.nodes.at(n.id);
    const bool mul = n.op == HG_OP_MULTIPLY;
    const bool rs = np.decision == HG_RESCALE_AFTER;
    const double s = ctx.default_scale;
    Value v;
    v.is_cipher = true;
    if (a.is_cipher && b.is_cipher) {
      const CtBatch& ca = a.cipher;
      const CtBatch& cb = b.cipher;
      require(ca.count == cb.count, "elementwise shape mismatch");
      if (mul) {
        require(rk_ != nullptr, "graph contains cipher-cipher products but no relin key");
        check_cc_mul(ca);
        check_cc_mul(cb);
        check_same_shape(ca, cb);
        v.cipher = do_relin(ctx, *rk_, &ca, &cb, 1, rs, s_);
        relins_ += ca.count;
        if (rs) rescales_ += ca.count;
      } else {
        check_same_shape(ca, cb);
        v.cipher.packing = ca.packing;
        v.cipher.scale = ca.scale;
        ensure(ctx, v.cipher, ca.count, 2, ca.level, s_);
        EwArgs e{};
        e.op = EwOp::AddCC;
        e.a = ca.data();
        e.b = cb.data();
        e.out = v.cipher.data();
        e.count = ca.count;
        e.polys_a = 2;
        e.polys_out = 2;
        e.level = ca.level;
        run_ew(ctx, e, s_);
      }
    } else {
      const CtBatch& x = a.is_cipher ? a.cipher : b.cipher;
      WeightTensor& c = *(a.is_cipher ? b.plain : a.plain);
      const bool broadcast = c.data.size() == 1;
      require(broadcast || c.data.size() == x.count, "elementwise shape mismatch");
      const float* cd = weight_dev(ctx, c, s_);
      const u32 L = x.level;
      v.cipher.packing = x.packing;
      if (mul) {
        check_scalar_encodable(ctx, c.max_abs, L, s);
        BufPtr res = ctx.alloc(static_cast<u64>(c.data.size()) * L * ctx.word_bytes(), s_);
        // residues laid out [value][limb]
        int r = encode_f32(ctx, cd, c.data.size(), 1, L, 1, L, s, res->ptr, s_);
        check_launch(r, "encode");
        v.cipher.scale = x.scale * s;
        ensure(ctx, v.cipher, x.count, 2, L, s_);
        EwArgs e{};
        e.op = EwOp::MulScalar;
        e.a = x.data();
        e.res = static_cast<const u32*>(res->ptr);
        e.per_element = broadcast ? 0 : 1;
        e.out = v.cipher.data();
        e.count = x.count;
        e.polys_a = 2;
        e.polys_out = 2;
        e.level = L;
        run_ew(ctx, e, s_);
        if (rs) {
          v.cipher = do_rescale(ctx, v.cipher, L - 1, s_);
          rescales_ += x.count;
        }
      } else {
        v.cipher.scale = x.scale;
        ensure(ctx, v.cipher, x.count, 2, L, s_);
        EwArgs e{};
        e.a = x.data();
        e.out = v.cipher.data();
        e.count = x.count;
        e.polys_a = 2;
        e.polys_out = 2;
        e.level = L;
        e.per_element = broadcast ? 0 : 1;
        BufPtr res;
        if (model_.packing == HG_PACKING_REAL) {
          check_scalar_encodable(ctx, c.max_abs, L, x.scale);
          res = ctx.alloc(static_cast<u64>(c.data.size()) * L * ctx.word_bytes(), s_);
          int r = encode_f32(ctx, cd, c.data.size(), 1, L, 1, L, x.scale, res->ptr, s_);
          check_launch(r, "encode");
          e.op = EwOp::AddScalar;
          e.res = static_cast<const u32*>(res->ptr);
        } else {
          std::vector<double> slots(c.data.size() * ctx.n);
          for (u64 i = 0; i < c.data.size(); ++i)
            for (u32 j = 0; j < ctx.n / 2; ++j) {
              slots[(i * ctx.n / 2 + j) * 2] = c.data[i];
              slots[(i * ctx.n / 2 + j) * 2 + 1] = c.data[i];
            }
          BufPtr ds = ctx.alloc(slots.size() * sizeof(double), s_);
          cuda_check(cudaMemcpyAsync(ds->ptr, slots.data(), slots.size() * sizeof(double), cudaMemcpyHostToDevice, s_),
                     "h2d");
          std::vector<unsigned long long> mant;
          std::vector<int> ex;
          res = encode_vectors_dev(ctx, static_cast<const double*>(ds->ptr), ctx.n / 2, c.data.size(), L, x.scale, s_,
                                   mant, ex);
          e.op = EwOp::AddVector;
          e.b = static_cast<const u32*>(res->ptr);
        }
        run_ew(ctx, e, s_);
      }
    }
    v.cipher.shape = model_.shapes.at(n.id);
    return v;
  }

  Value eval_nonlinear(const Node& n, std::map<std::string, Value>& values, u32 layer_seq, hg_exec_stats* stats) {
    require(provider_ != nullptr, "graph contains " + n.id + " but no nonlinearity provider is attached");
    const Context& ctx = *ctx_;
    const CtBatch& x = values.at(n.inputs[0]).cipher;
    const auto& out_shape = model_.shapes.at(n.id);
    hg_tensor req;
    req.ctx = ctx_;
    u32 window = 1;
    if (n.op == HG_OP_RELU) {
      req.b = x;
    } else {
      // one window-sized group per output element (henet/graph.hpp:1072-1094): gather on device
      const u32 stride = n.attrs.pool_stride ? n.attrs.pool_stride : n.attrs.window;
      const u32 win = n.attrs.window;
      window = win * win;
      const u32 C = out_shape[0], oh = out_shape[1], ow = out_shape[2];
      const u32 ihh = x.shape[1], iww = x.shape[2];
      CtBatch g;
      g.packing = x.packing;
      g.scale = x.scale;
      ensure(ctx, g, static_cast<u64>(C) * oh * ow * window, 2, x.level, s_);
      const u64 ct_bytes = 2ull * x.level * ctx.n * ctx.word_bytes();
      u64 o = 0;
      for (u32 c = 0; c < C; ++c)
        for (u32 y = 0; y < oh; ++y)
          for (u32 xo = 0; xo < ow; ++xo)
            for (u32 ky = 0; ky < win; ++ky)
              for (u32 kx = 0; kx < win; ++kx) {
                const u64 idx = (static_cast<u64>(c) * ihh + (y * stride + ky)) * iww + (xo * stride + kx);
                cuda_check(cudaMemcpyAsync(static_cast<char*>(g.buf->ptr) + o * ct_bytes,
                                           static_cast<const char*>(x.buf->ptr) + idx * ct_bytes, ct_bytes,
                                           cudaMemcpyDeviceToDevice, s_),
                           "gather");
                ++o;
              }
      req.b = g;
    }
    hg_tensor resp;
    resp.ctx = ctx_;
    resp.b.packing = x.packing;
    resp.b.scale = ctx.default_scale;
    static const bool trace = getenv("HG_REFRESH_TRACE") != nullptr;
    const auto t_a = std::chrono::steady_clock::now();
    ensure(ctx, resp.b, elem_count(out_shape), 2, static_cast<u32>(ctx.chain_len()), s_);
    const auto t_b = std::chrono::steady_clock::now();
    cuda_check(cudaStreamSynchronize(s_), "nonlinearity");
    if (trace)
      std::fprintf(stderr, "nonlinearity %s: response alloc %.2f ms, sync %.2f ms\n", n.id.c_str(),
                   std::chrono::duration<double, std::milli>(t_b - t_a).count(),
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_b).count());
    const int rc = provider_(user_, n.op == HG_OP_RELU ? HG_NONLIN_RELU : HG_NONLIN_MAXPOOL, window, layer_seq, &req, &resp);
    if (rc != 0) throw Error(HG_ERR_VALIDATION, "nonlinearity provider failed: " + g_last_error);
    require(resp.b.count == elem_count(out_shape), "provider returned the wrong element count");
    require(resp.b.level == ctx.chain_len(), "provider must refresh to the top level");
    if (stats) stats->nonlin_elements += req.b.count;
    Value v;
    v.is_cipher = true;
    v.cipher = resp.b;
    v.cipher.shape = out_shape;
    return v;
  }

  std::shared_ptr<Context> ctx_;
  Model& model_;
  const Plan& plan_;
  const RelinKeyDev* rk_;
  hg_nonlin_fn provider_;
  void* user_;
  cudaStream_t s_;
  bool timing_;
  bool keep_ = false;  // model_.keep_encodings, read once per execute under the model mutex
  u64 rescales_ = 0, relins_ = 0;
  u64 launches0_ = launches_total();  // kernel launches are counted process-wide
};

}  // namespace hg

// ===========================================================================
// C ABI
// ===========================================================================
using namespace hg;

extern "C" {

const char* hg_last_error(void) { return g_last_error.c_str(); }
int hg_abi_version(void) { return HG_ABI_VERSION; }

int hg_ctx_create(uint32_t poly_degree, const uint64_t* chain, uint32_t chain_len, uint64_t special,
                  double default_scale, int device, hg_ctx** out) {
  return guard([&] {
    require(out != nullptr && chain != nullptr, "null argument");
    auto c = make_context(poly_degree, chain, chain_len, special, default_scale, device);
    *out = new hg_ctx{c, {}};
  });
}

void hg_ctx_destroy(hg_ctx* ctx) { delete ctx; }

int hg_ctx_ntt_root(const hg_ctx* ctx, uint32_t i, uint64_t* root) {
  return guard([&] {
    require(ctx && root, "null argument");
    require(i < ctx->c->roots.size(), "basis index out of range");
    *root = ctx->c->roots[i];
  });
}

void* hg_ctx_stream(hg_ctx* ctx) { return ctx ? ctx->c->core->stream : nullptr; }

int hg_ctx_synchronize(hg_ctx* ctx) {
  return guard([&] { cuda_check(cudaStreamSynchronize(ctx->c->core->stream), "synchronize"); });
}

uint64_t hg_ctx_launch_count(const hg_ctx* ctx) { return ctx ? hg::launches_total() : 0; }

int hg_tensor_create(hg_ctx* ctx, uint64_t count, uint32_t polys, uint32_t level, double scale, int packing,
                     hg_tensor** out) {
  return guard([&] {
    require(ctx && out, "null argument");
    require(polys == 2 || polys == 3, "ciphertext must have 2 or 3 polynomials");
    require(level >= 1 && level <= ctx->c->chain_len(), "level outside the context chain");
    require(packing == HG_PACKING_REAL || packing == HG_PACKING_COMPLEX, "unknown packing mode");
    auto* t = new hg_tensor;
    t->ctx = ctx->c;
    t->b.scale = scale;
    t->b.packing = packing;
    ensure(*ctx->c, t->b, count, polys, level, nullptr);
    t->b.shape = {static_cast<u32>(count)};
    *out = t;
  });
}

void hg_tensor_destroy(hg_tensor* t) { delete t; }

int hg_tensor_info(const hg_tensor* t, uint64_t* count, uint32_t* polys, uint32_t* level, double* scale,
                   int* packing) {
  return guard([&] {
    require(t != nullptr, "null tensor");
    if (count) *count = t->b.count;
    if (polys) *polys = t->b.polys;
    if (level) *level = t->b.level;
    if (scale) *scale = t->b.scale;
    if (packing) *packing = t->b.packing;
  });
}

int hg_tensor_set_scale(hg_tensor* t, double scale) {
  return guard([&] { t->b.scale = scale; });
}

int hg_tensor_set_shape(hg_tensor* t, const uint32_t* dims, uint32_t ndims) {
  return guard([&] {
    std::vector<u32> d(dims, dims + ndims);
    require(elem_count(d) == t->b.count, "shape does not match the element count");
    t->b.shape = d;
  });
}

int hg_tensor_get_shape(const hg_tensor* t, uint32_t* dims, uint32_t* ndims) {
  return guard([&] {
    require(*ndims >= t->b.shape.size(), "shape buffer too small");
    for (size_t i = 0; i < t->b.shape.size(); ++i) dims[i] = t->b.shape[i];
    *ndims = static_cast<uint32_t>(t->b.shape.size());
  });
}

int hg_tensor_upload(hg_tensor* t, const uint64_t* words, void* stream) {
  return guard([&] {
    const Context& ctx = *t->ctx;
    cudaStream_t s = ctx.pick(stream);
    const u64 n = t->b.words(ctx.n);
    if (!ctx.wide && host_narrow_enabled()) {
      // PCIe and the host packers both bound this path: the last ~15% of the ciphertexts
      // cross as raw u64 and are narrowed on the GPU while the host packs the rest
      const u64 per_ct = static_cast<u64>(t->b.polys) * t->b.level * ctx.n;
      const u64 dcts = static_cast<u64>(static_cast<double>(t->b.count) * upload_direct_fraction());
      DirectShare ds{dcts * per_ct, nullptr, nullptr, &ctx.basis};
      if (ds.words) {
        const size_t need = ds.words * 8 + sizeof(int);
        if (!t->stage || t->stage->bytes < need) {
          t->stage = ctx.alloc(need, ctx.core->stream);
          cuda_check(cudaStreamSynchronize(ctx.core->stream), "upload staging");
        }
        ds.stage = static_cast<u64*>(t->stage->ptr);
        ds.bad = reinterpret_cast<int*>(static_cast<char*>(t->stage->ptr) + ds.words * 8);
      }
      require(host_narrow_upload(ctx.core->device, words, t->b.data(), n - ds.words, t->b.level, ctx.n,
                                 ctx.chain.data(), s, nullptr, 0, &ds),
              "residue out of range");
      return;
    }
    int r;
    const size_t need = (ctx.wide ? 0 : n * 8) + sizeof(int);
    if (!t->stage || t->stage->bytes < need) {
      // allocated on the context's own stream (it outlives any caller stream), then ready
      t->stage = ctx.alloc(need, ctx.core->stream);
      cuda_check(cudaStreamSynchronize(ctx.core->stream), "upload staging");
    }
    BufPtr stage = t->stage;
    int* bad = reinterpret_cast<int*>(static_cast<char*>(stage->ptr) + (ctx.wide ? 0 : n * 8));
    cuda_check(cudaMemsetAsync(bad, 0, sizeof(int), s), "memset");
    if (ctx.wide) {
      cuda_check(cudaMemcpyAsync(t->b.data64(), words, n * 8, cudaMemcpyHostToDevice, s), "h2d");
      r = launch_validate_w(t->b.data64(), n, t->b.level, ctx.n, ctx.basisw, bad, s);
    } else {
      cuda_check(cudaMemcpyAsync(stage->ptr, words, n * 8, cudaMemcpyHostToDevice, s), "h2d");
      r = launch_narrow(static_cast<const u64*>(stage->ptr), t->b.data(), n, t->b.level, ctx.n, ctx.basis, bad, s);
    }
    check_launch(r, "narrow");
    int hbad = 0;
    cuda_check(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
    cuda_check(cudaStreamSynchronize(s), "upload");
    require(hbad == 0, "residue out of range");
  });
}

int hg_tensor_download(const hg_tensor* t, uint64_t* words, void* stream) {
  return guard([&] {
    const Context& ctx = *t->ctx;
    cudaStream_t s = ctx.pick(stream);
    const u64 n = t->b.words(ctx.n);
    if (ctx.wide) {
      cuda_check(cudaMemcpyAsync(words, t->b.data64(), n * 8, cudaMemcpyDeviceToHost, s), "d2h");
    } else {
      BufPtr stage = ctx.alloc(n * 8, s);
      const int r = launch_widen(t->b.data(), static_cast<u64*>(stage->ptr), n, s);
      check_launch(r, "widen");
      cuda_check(cudaMemcpyAsync(words, stage->ptr, n * 8, cudaMemcpyDeviceToHost, s), "d2h");
    }
    cuda_check(cudaStreamSynchronize(s), "download");
  });
}

int hg_tensor_assign(hg_tensor* dst, const hg_tensor* src) {
  return guard([&] {
    require(dst != nullptr && src != nullptr, "null argument");
    require(dst->ctx == src->ctx, "tensors belong to different contexts");
    dst->b = src->b;  // shares the device buffer (reference counted)
  });
}

int hg_tensor_upload_segments(hg_tensor* t, const uint64_t* const* segs, void* stream) {
  return guard([&] {
    require(t != nullptr && segs != nullptr, "null argument");
    const Context& ctx = *t->ctx;
    cudaStream_t s = ctx.pick(stream);
    const u64 seg_words = static_cast<u64>(t->b.level) * ctx.n;
    const u64 nseg = t->b.count * t->b.polys;
    const u64 n = nseg * seg_words;
    if (!ctx.wide && host_narrow_enabled()) {
      // the packer threads read each segment in place (as hg_tensor_deserialize does)
      require(host_narrow_upload(ctx.core->device, nullptr, t->b.data(), n, t->b.level, ctx.n, ctx.chain.data(), s,
                                 reinterpret_cast<const uint8_t* const*>(segs), seg_words),
              "residue out of range");
      return;
    }
    const size_t need = (ctx.wide ? 0 : n * 8) + sizeof(int);
    if (!t->stage || t->stage->bytes < need) {
      t->stage = ctx.alloc(need, ctx.core->stream);
      cuda_check(cudaStreamSynchronize(ctx.core->stream), "upload staging");
    }
    BufPtr stage = t->stage;
    int* bad = reinterpret_cast<int*>(static_cast<char*>(stage->ptr) + (ctx.wide ? 0 : n * 8));
    cuda_check(cudaMemsetAsync(bad, 0, sizeof(int), s), "memset");
    u64* dst = ctx.wide ? t->b.data64() : static_cast<u64*>(stage->ptr);
    for (u64 i = 0; i < nseg; ++i)
      cuda_check(cudaMemcpyAsync(dst + i * seg_words, segs[i], seg_words * 8, cudaMemcpyHostToDevice, s), "h2d");
    const int r = ctx.wide ? launch_validate_w(t->b.data64(), n, t->b.level, ctx.n, ctx.basisw, bad, s)
                           : launch_narrow(dst, t->b.data(), n, t->b.level, ctx.n, ctx.basis, bad, s);
    check_launch(r, "narrow");
    int hbad = 0;
    cuda_check(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s), "d2h");
    cuda_check(cudaStreamSynchronize(s), "upload");
    require(hbad == 0, "residue out of range");
  });
}

int hg_tensor_download_segments(const hg_tensor* t, uint64_t* const* segs, void* stream) {
  return guard([&] {
    require(t != nullptr && segs != nullptr, "null argument");
    const Context& ctx = *t->ctx;
    cudaStream_t s = ctx.pick(stream);
    const u64 seg_words = static_cast<u64>(t->b.level) * ctx.n;
    const u64 nseg = t->b.count * t->b.polys;
    const u64 n = nseg * seg_words;
    BufPtr stage;
    const u64* src = ctx.wide ? t->b.data64() : nullptr;
    if (!ctx.wide) {
      stage = ctx.alloc(n * 8, s);
      check_launch(launch_widen(t->b.data(), static_cast<u64*>(stage->ptr), n, s), "widen");
      src = static_cast<const u64*>(stage->ptr);
    }
    for (u64 i = 0; i < nseg; ++i)
      cuda_check(cudaMemcpyAsync(segs[i], src + i * seg_words, seg_words * 8, cudaMemcpyDeviceToHost, s), "d2h");
    cuda_check(cudaStreamSynchronize(s), "download");
  });
}

int hg_tensor_upload_u32(hg_tensor* t, const uint32_t* words, void* stream) {
  return guard([&] {
    const Context& ctx = *t->ctx;
    if (ctx.wide) throw Error(HG_ERR_UNSUPPORTED, "u32 residues: this context stores u64 words (primes >= 2^30)");
    cuda_check(cudaMemcpyAsync(t->b.data(), words, t->b.words(ctx.n) * 4, cudaMemcpyHostToDevice, ctx.pick(stream)),
               "h2d");
  });
}

int hg_tensor_download_u32(const hg_tensor* t, uint32_t* words, void* stream) {
  return guard([&] {
    const Context& ctx = *t->ctx;
    if (ctx.wide) throw Error(HG_ERR_UNSUPPORTED, "u32 residues: this context stores u64 words (primes >= 2^30)");
    cudaStream_t s = ctx.pick(stream);
    cuda_check(cudaMemcpyAsync(words, t->b.data(), t->b.words(ctx.n) * 4, cudaMemcpyDeviceToHost, s), "d2h");
    cuda_check(cudaStreamSynchronize(s), "download");
  });
}

void* hg_tensor_device_ptr(hg_tensor* t) { return t ? t->b.data() : nullptr; }
uint64_t hg_tensor_words(const hg_tensor* t) { return t ? t->b.words(t->ctx->n) : 0; }
uint32_t hg_tensor_word_bytes(const hg_tensor* t) { return t ? (t->ctx->wide ? 8u : 4u) : 0u; }

int hg_relin_key_upload(hg_ctx* ctx, const uint64_t* words, uint64_t n_words, hg_relin_key** out) {
  return guard([&] {
    const Context& c = *ctx->c;
    require(c.has_special, "relinearization keys need a special prime (not present in these parameters)");
    const u64 L = c.chain_len(), n = c.n;
    require(n_words == L * 2 * (L + 1) * n, "malformed relinearization key");
    if (c.wide) {
      // u64 contexts: the serialized words as they are ([j][c][t][N]), range-checked
      for (u64 j = 0; j < L; ++j)
        for (u64 p = 0; p < 2; ++p)
          for (u64 t = 0; t <= L; ++t) {
            const u64 q = c.basis_mod(t);
            const u64 base = ((j * 2 + p) * (L + 1) + t) * n;
            for (u64 i = 0; i < n; ++i) require(words[base + i] < q, "residue out of range");
          }
      auto* rk = new hg_relin_key;
      rk->ctx = ctx->c;
      rk->k.chain_len = static_cast<u32>(L);
      rk->k.key = c.alloc(n_words * 8, nullptr);
      cuda_check(cudaMemcpyAsync(rk->k.key->ptr, words, n_words * 8, cudaMemcpyHostToDevice, c.core->stream), "h2d");
      cuda_check(cudaStreamSynchronize(c.core->stream), "relin key upload");
      *out = rk;
      return;
    }
    // device layout (hg::kKeyShoup): (value, shoup) pairs, or values only
    const size_t esz = kKeyShoup ? sizeof(uint2) : sizeof(u32);
    std::vector<unsigned char> k(n_words * esz);
    for (u64 j = 0; j < L; ++j)
      for (u64 p = 0; p < 2; ++p)
        for (u64 t = 0; t <= L; ++t) {
          const u64 q = c.basis_mod(t);
          const u64 base = ((j * 2 + p) * (L + 1) + t) * n;
          // chain columns carry the mod-down's P^-1 (hg::kKeyPinv)
          const u64 fold = (kKeyPinv && t < L) ? nt::inv(c.special % q, q) : 1;
          for (u64 i = 0; i < n; ++i) {
            require(words[base + i] < q, "residue out of range");
            const u64 w = static_cast<u64>(static_cast<nt::u128>(words[base + i]) * fold % q);
            if (kKeyShoup)
              reinterpret_cast<uint2*>(k.data())[base + i] = make_uint2(static_cast<u32>(w), nt::shoup(w, q));
            else
              reinterpret_cast<u32*>(k.data())[base + i] = static_cast<u32>(w);
          }
        }
    auto* rk = new hg_relin_key;
    rk->ctx = ctx->c;
    rk->k.chain_len = static_cast<u32>(L);
    rk->k.key = c.alloc(k.size(), nullptr);
    cuda_check(cudaMemcpyAsync(rk->k.key->ptr, k.data(), k.size(), cudaMemcpyHostToDevice, c.core->stream), "h2d");
    cuda_check(cudaStreamSynchronize(c.core->stream), "relin key upload");
    *out = rk;
  });
}

void hg_relin_key_destroy(hg_relin_key* rk) { delete rk; }

int hg_add_ct_ct(hg_ctx* ctx, const hg_tensor* a, const hg_tensor* b, hg_tensor* out, void* stream) {
  return guard([&] {
    const Context& c = *ctx->c;
    cudaStream_t s = c.pick(stream);
    check_same_shape(a->b, b->b);
    CtBatch o;
    o.packing = a->b.packing;
    o.scale = a->b.scale;
    o.shape = a->b.shape;
    ensure(c, o, a->b.count, a->b.polys, a->b.level, s);
    EwArgs e{};
    e.op = EwOp::AddCC;
    e.a = a->b.data();
    e.b = b->b.data();
    e.out = o.data();
    e.count = a->b.count;
    e.polys_a = a->b.polys;
    e.polys_out = a->b.polys;
    e.level = a->b.level;
    run_ew(c, e, s);
    out->b = o;
  });
}

static BufPtr upload_residues(const Context& c, const hg_tensor* ct, const uint64_t* residues, int per_element,
                              cudaStream_t s) {
  const u64 nvals = (per_element ? ct->b.count : 1) * ct->b.level;
  for (u64 i = 0; i < nvals; ++i) require(residues[i] < c.chain[i % ct->b.level], "residue out of range");
  BufPtr d = c.alloc(nvals * c.word_bytes(), s);
  if (c.wide) {
    cuda_check(cudaMemcpyAsync(d->ptr, residues, nvals * 8, cudaMemcpyHostToDevice, s), "h2d");
  } else {
    std::vector<u32> r(residues, residues + nvals);
    cuda_check(cudaMemcpyAsync(d->ptr, r.data(), nvals * 4, cudaMemcpyHostToDevice, s), "h2d");
  }
  cuda_check(cudaStreamSynchronize(s), "h2d");
  return d;
}

int hg_mul_ct_pt_scalar(hg_ctx* ctx, const hg_tensor* ct, const uint64_t* residues, int per_element, double pt_scale,
                        hg_tensor* out, void* stream) {
  return guard([&] {
    const Context& c = *ctx->c;
    cudaStream_t s = c.pick(stream);
    BufPtr r = upload_residues(c, ct, residues, per_element, s);
    CtBatch o;
    o.packing = ct->b.packing;
    o.scale = ct->b.scale * pt_scale;
    o.shape = ct->b.shape;
    ensure(c, o, ct->b.count, ct->b.polys, ct->b.level, s);
    EwArgs e{};
    e.op = EwOp::MulScalar;
    e.a = ct->b.data();
    e.res = static_cast<const u32*>(r->ptr);
    e.per_element = per_element;
    e.out = o.data();
    e.count = ct->b.count;
    e.polys_a = ct->b.polys;
    e.polys_out = ct->b.polys;
    e.level = ct->b.level;
    run_ew(c, e, s);
    out->b = o;
  });
}

int hg_add_ct_pt_scalar(hg_ctx* ctx, const hg_tensor* ct, const uint64_t* residues, int per_element, double pt_scale,
                        hg_tensor* out, void* stream) {
  return guard([&] {
    const Context& c = *ctx->c;
    cudaStream_t s = c.pick(stream);
    require(scales_match(ct->b.scale, pt_scale), "ciphertext/plaintext scale mismatch");
    BufPtr r = upload_residues(c, ct, residues, per_element, s);
    CtBatch o;
    o.packing = ct->b.packing;
    o.scale = ct->b.scale;
    o.shape = ct->b.shape;
    ensure(c, o, ct->b.count, ct->b.polys, ct->b.level, s);
    EwArgs e{};
    e.op = EwOp::AddScalar;
    e.a = ct->b.data();
    e.res = static_cast<const u32*>(r->ptr);
    e.per_element = per_element;
    e.out = o.data();
    e.count = ct->b.count;
    e.polys_a = ct->b.polys;
    e.polys_out = ct->b.polys;
    e.level = ct->b.level;
    run_ew(c, e, s);
    out->b = o;
  });
}

int hg_add_ct_pt_vector(hg_ctx* ctx, const hg_tensor* ct, const uint64_t* pt_words, int per_element, double pt_scale,
                        hg_tensor* out, void* stream) {
  return guard([&] {
    const Context& c = *ctx->c;
    cudaStream_t s = c.pick(stream);
    require(scales_match(ct->b.scale, pt_scale), "ciphertext/plaintext scale mismatch");
    const u64 L = ct->b.level, n = c.n;
    const u64 nw = (per_element ? ct->b.count : 1) * L * n;
    for (u64 i = 0; i < nw; ++i) require(pt_words[i] < c.chain[(i / n) % L], "residue out of range");
    BufPtr d = c.alloc(nw * c.word_bytes(), s);
    std::vector<u32> w;
    if (c.wide) {
      cuda_check(cudaMemcpyAsync(d->ptr, pt_words, nw * 8, cudaMemcpyHostToDevice, s), "h2d");
    } else {
      w.assign(pt_words, pt_words + nw);
      cuda_check(cudaMemcpyAsync(d->ptr, w.data(), nw * 4, cudaMemcpyHostToDevice, s), "h2d");
    }
    CtBatch o;
    o.packing = ct->b.packing;
    o.scale = ct->b.scale;
    o.shape = ct->b.shape;
    ensure(c, o, ct->b.count, ct->b.polys, ct->b.level, s);
    EwArgs e{};
    e.op = EwOp::AddVector;
    e.a = ct->b.data();
    e.b = static_cast<const u32*>(d->ptr);
    e.per_element = per_element;
    e.out = o.data();
    e.count = ct->b.count;
    e.polys_a = ct->b.polys;
    e.polys_out = ct->b.polys;
    e.level = ct->b.level;
    run_ew(c, e, s);
    cuda_check(cudaStreamSynchronize(s), "add_ct_pt_vector");
    out->b = o;
  });
}

static void tensor_op(hg_ctx* ctx, const hg_tensor* a, const hg_tensor* b, hg_tensor* out, void* stream) {
  const Context& c = *ctx->c;
  cudaStream_t s = c.pick(stream);
  check_cc_mul(a->b);
  check_cc_mul(b->b);
  if (a != b) check_same_shape(a->b, b->b);
  CtBatch o;
  o.packing = a->b.packing;
  o.scale = a->b.scale * b->b.scale;
  o.shape = a->b.shape;
  ensure(c, o, a->b.count, 3, a->b.level, s);
  EwArgs e{};
  e.op = EwOp::Tensor;
  e.a = a->b.data();
  e.b = b->b.data();
  e.out = o.data();
  e.count = a->b.count;
  e.polys_a = 2;
  e.polys_out = 3;
  e.level = a->b.level;
  run_ew(c, e, s);
  out->b = o;
}

int hg_square(hg_ctx* ctx, const hg_tensor* ct, hg_tensor* out, void* stream) {
  return guard([&] { tensor_op(ctx, ct, ct, out, stream); });
}

int hg_mul_ct_ct(hg_ctx* ctx, const hg_tensor* a, const hg_tensor* b, hg_tensor* out, void* stream) {
  return guard([&] { tensor_op(ctx, a, b, out, stream); });
}

int hg_relinearize(hg_ctx* ctx, const hg_tensor* ct, const hg_relin_key* rk, hg_tensor* out, void* stream) {
  return guard([&] {
    require(ct->b.polys == 3, "relinearize expects a size-3 ciphertext");
    CtBatch o = do_relin(*ctx->c, rk->k, &ct->b, nullptr, 0, false, ctx->c->pick(stream));
    o.shape = ct->b.shape;
    out->b = o;
  });
}

int hg_square_relin(hg_ctx* ctx, const hg_tensor* ct, const hg_relin_key* rk, int rescale, hg_tensor* out,
                    void* stream) {
  return guard([&] {
    check_cc_mul(ct->b);
    CtBatch o = do_relin(*ctx->c, rk->k, &ct->b, &ct->b, 1, rescale != 0, ctx->c->pick(stream));
    o.shape = ct->b.shape;
    out->b = o;
  });
}

int hg_rescale(hg_ctx* ctx, const hg_tensor* ct, uint32_t target_level, hg_tensor* out, void* stream) {
  return guard([&] {
    CtBatch o = do_rescale(*ctx->c, ct->b, target_level, ctx->c->pick(stream));
    o.shape = ct->b.shape;
    out->b = o;
  });
}

int hg_ntt_forward(hg_ctx* ctx, hg_tensor* t, void* stream) {
  return guard([&] {
    const Context& c = *ctx->c;
    const u64 rows = t->b.count * t->b.polys * t->b.level;
    const int r = c.wide ? launch_ntt_w(static_cast<int>(c.logn), t->b.data64(), rows, t->b.level, false, c.basisw,
                                        c.pick(stream))
                         : launch_ntt(static_cast<int>(c.logn), t->b.data(), rows, t->b.level, false, c.basis,
                                      c.pick(stream));
    check_launch(r, "ntt");
  });
}

int hg_ntt_inverse(hg_ctx* ctx, hg_tensor* t, void* stream) {
  return guard([&] {
    const Context& c = *ctx->c;
    const u64 rows = t->b.count * t->b.polys * t->b.level;
    const int r = c.wide ? launch_ntt_w(static_cast<int>(c.logn), t->b.data64(), rows, t->b.level, true, c.basisw,
                                        c.pick(stream))
                         : launch_ntt(static_cast<int>(c.logn), t->b.data(), rows, t->b.level, true, c.basis,
                                      c.pick(stream));
    check_launch(r, "intt");
  });
}

int hg_encode_scalars(hg_ctx* ctx, const double* values, uint64_t count, uint32_t level, double scale,
                      uint64_t* out_residues) {
  return guard([&] {
    const Context& c = *ctx->c;
    cudaStream_t s = c.core->stream;
    double mx = 0;
    for (u64 i = 0; i < count; ++i) mx = std::max(mx, std::fabs(values[i]));
    check_scalar_encodable(c, mx, level, scale);
    BufPtr dv = c.alloc(count * 8, s);
    BufPtr dr = c.alloc(count * level * c.word_bytes(), s);
    cuda_check(cudaMemcpyAsync(dv->ptr, values, count * 8, cudaMemcpyHostToDevice, s), "h2d");
    const int r = c.wide ? launch_encode_scalars_w_f64(static_cast<const double*>(dv->ptr), count, 1, level, 1, level,
                                                       scale, static_cast<u64*>(dr->ptr), c.basisw, s)
                         : launch_encode_scalars_f64(static_cast<const double*>(dv->ptr), count, 1, level, 1, level,
                                                     scale, static_cast<u32*>(dr->ptr), c.basis, s);
    check_launch(r, "encode_scalars");
    if (c.wide) {
      cuda_check(cudaMemcpyAsync(out_residues, dr->ptr, count * level * 8, cudaMemcpyDeviceToHost, s), "d2h");
      cuda_check(cudaStreamSynchronize(s), "encode_scalars");
    } else {
      std::vector<u32> h(count * level);
      cuda_check(cudaMemcpyAsync(h.data(), dr->ptr, h.size() * 4, cudaMemcpyDeviceToHost, s), "d2h");
      cuda_check(cudaStreamSynchronize(s), "encode_scalars");
      for (u64 i = 0; i < h.size(); ++i) out_residues[i] = h[i];
    }
  });
}

int hg_encode_vector(hg_ctx* ctx, const double* slots_re_im, uint32_t n_slots, uint64_t count, uint32_t level,
                     double scale, uint64_t* out_words) {
  return guard([&] {
    const Context& c = *ctx->c;
    cudaStream_t s = c.core->stream;
    BufPtr ds = c.alloc(count * n_slots * 2 * sizeof(double) + 16, s);
    cuda_check(cudaMemcpyAsync(ds->ptr, slots_re_im, count * n_slots * 2 * sizeof(double), cudaMemcpyHostToDevice, s),
               "h2d");
    std::vector<unsigned long long> mant;
    std::vector<int> ex;
    BufPtr pt = encode_vectors_dev(c, static_cast<const double*>(ds->ptr), n_slots, count, level, scale, s, mant, ex);
    const u64 nw = count * level * static_cast<u64>(c.n);
    if (c.wide) {
      cuda_check(cudaMemcpyAsync(out_words, pt->ptr, nw * 8, cudaMemcpyDeviceToHost, s), "d2h");
      cuda_check(cudaStreamSynchronize(s), "encode_vector");
    } else {
      std::vector<u32> h(nw);
      cuda_check(cudaMemcpyAsync(h.data(), pt->ptr, nw * 4, cudaMemcpyDeviceToHost, s), "d2h");
      cuda_check(cudaStreamSynchronize(s), "encode_vector");
      for (u64 i = 0; i < nw; ++i) out_words[i] = h[i];
    }
  });
}

int hg_model_create(int packing, hg_model** out) {
  return guard([&] {
    require(packing == HG_PACKING_REAL || packing == HG_PACKING_COMPLEX, "unknown packing mode");
    auto* m = new hg_model;
    m->m.packing = packing;
    *out = m;
  });
}

void hg_model_destroy(hg_model* m) { delete m; }

int hg_model_add_weight(hg_model* m, const char* name, const uint32_t* dims, uint32_t ndims, const float* data) {
  return guard([&] {
    WeightTensor w;
    w.dims.assign(dims, dims + ndims);
    const u64 n = elem_count(w.dims);
    w.data.assign(data, data + n);
    for (float v : w.data) w.max_abs = std::max(w.max_abs, std::fabs(v));
    m->m.weights[name] = std::move(w);
    m->m.finalized = false;
  });
}

int hg_model_add_node(hg_model* m, const hg_node_desc* d) {
  return guard([&] {
    require(d && d->id, "null node");
    require(d->op >= HG_OP_INPUT && d->op <= HG_OP_OUTPUT, "unknown op");
    Node n;
    n.id = d->id;
    n.op = d->op;
    for (u32 i = 0; i < d->n_inputs; ++i) n.inputs.emplace_back(d->inputs[i]);
    if (d->shape) n.attrs.shape.assign(d->shape, d->shape + d->shape_len);
    n.attrs.stride = d->stride ? d->stride : 1;
    n.attrs.window = d->window;
    n.attrs.filters = d->filters;
    n.attrs.pool_stride = d->pool_stride;
    for (int i = 0; i < 4; ++i) n.attrs.pad[i] = d->pad[i];
    if (d->weight_ref) n.weight_ref = d->weight_ref;
    if (d->bias_ref) n.bias_ref = d->bias_ref;
    require(!m->m.index.count(n.id), "duplicate node id: " + n.id);
    m->m.index.emplace(n.id, m->m.nodes.size());
    m->m.nodes.push_back(std::move(n));
    m->m.finalized = false;
  });
}

int hg_model_finalize(hg_model* m) {
  return guard([&] { finalize_model(m->m); });
}

int hg_model_node_count(const hg_model* m, uint32_t* n) {
  return guard([&] { *n = static_cast<uint32_t>(m->m.nodes.size()); });
}

int hg_model_shape(const hg_model* m, const char* id, uint32_t* dims, uint32_t* ndims) {
  return guard([&] {
    auto it = m->m.shapes.find(id);
    require(it != m->m.shapes.end(), "unknown node id");
    require(*ndims >= it->second.size(), "shape buffer too small");
    for (size_t i = 0; i < it->second.size(); ++i) dims[i] = it->second[i];
    *ndims = static_cast<uint32_t>(it->second.size());
  });
}

int hg_plan_rescaling(const hg_ctx* ctx, const hg_model* m, int mode, hg_plan** out) {
  return guard([&] {
    Plan p = plan_rescaling(*ctx->c, m->m, mode);
    *out = new hg_plan{std::move(p)};
  });
}

int hg_plan_rescaling_params(const uint64_t* chain, uint32_t chain_len, double default_scale, const hg_model* m,
                             int mode, hg_plan** out) {
  return guard([&] {
    require(chain && chain_len >= 1, "modulus chain must be non-empty");
    Context c;  // host-side fields only: the planner needs no device
    c.chain.assign(chain, chain + chain_len);
    c.default_scale = default_scale;
    long double acc = 1.0L;
    c.modulus_products.push_back(acc);
    for (u64 q : c.chain) {
      acc *= static_cast<long double>(q);
      c.modulus_products.push_back(acc);
    }
    Plan p = plan_rescaling(c, m->m, mode);
    *out = new hg_plan{std::move(p)};
  });
}

int hg_plan_create(int mode, uint64_t planned, hg_plan** out) {
  return guard([&] {
    auto* p = new hg_plan;
    p->p.mode = mode;
    p->p.planned_rescale_ops = planned;
    *out = p;
  });
}

int hg_plan_set_node(hg_plan* p, const char* id, int decision, uint32_t level_in, uint32_t level_out, double scale_out) {
  return guard([&] {
    NodePlan np;
    np.decision = decision;
    np.level_in = level_in;
    np.level_out = level_out;
    np.scale_out = scale_out;
    p->p.nodes[id] = np;
  });
}

int hg_plan_get_node(const hg_plan* p, const char* id, int* decision, uint32_t* level_in, uint32_t* level_out,
                     double* scale_out) {
  return guard([&] {
    auto it = p->p.nodes.find(id);
    require(it != p->p.nodes.end(), "unknown node id");
    if (decision) *decision = it->second.decision;
    if (level_in) *level_in = it->second.level_in;
    if (level_out) *level_out = it->second.level_out;
    if (scale_out) *scale_out = it->second.scale_out;
  });
}

uint64_t hg_plan_planned_rescales(const hg_plan* p) { return p ? p->p.planned_rescale_ops : 0; }
void hg_plan_destroy(hg_plan* p) { delete p; }

int hg_execute(hg_ctx* ctx, const hg_model* m, const hg_plan* plan, const hg_tensor* input, const hg_relin_key* rk,
               hg_nonlin_fn provider, void* provider_user, hg_tensor** output, hg_exec_stats* stats, void* stream) {
  return guard([&] {
    require(ctx && m && plan && input && output, "null argument");
    if (stats) *stats = hg_exec_stats{};
    cudaStream_t s = ctx->c->pick(stream);
    const bool timing = getenv("HG_NODE_TIMING") != nullptr;
    Executor ex(ctx->c, const_cast<hg_model*>(m)->m, plan->p, rk ? &rk->k : nullptr, provider, provider_user, s, timing);
    CtBatch out = ex.run(input->b, stats, timing ? &ctx->last_node_ms : nullptr);
    auto* t = new hg_tensor;
    t->ctx = ctx->c;
    t->b = std::move(out);
    *output = t;
  });
}

int hg_bench_int_peak(int device, int kind, double* ops_per_s) {
  return guard([&] {
    *ops_per_s = kind == 4 ? bench_tc_i8_peak(device) : bench_int_peak(device, kind);
    cuda_check(cudaGetLastError(), "imad probe");
  });
}

int hg_prof_enable(int on) {
  return guard([&] { prof_enable(on != 0); });
}

int hg_prof_report(char* buf, uint64_t cap) {
  return guard([&] {
    const std::string r = prof_report();
    require(r.size() + 1 <= cap, "report buffer too small");
    std::memcpy(buf, r.c_str(), r.size() + 1);
  });
}

int hg_last_upload_h2d_bytes(uint64_t* bytes) {
  return guard([&] {
    require(bytes != nullptr, "null argument");
    *bytes = g_last_upload_h2d.load();
  });
}

int hg_last_exec_layer_count(uint32_t* n) {
  return guard([&] {
    require(n != nullptr, "null argument");
    *n = static_cast<uint32_t>(g_last_layers.size());
  });
}

int hg_last_exec_layer(uint32_t i, const char** id, double* ms) {
  return guard([&] {
    require(i < g_last_layers.size() && id && ms, "layer index out of range");
    *id = g_last_layers[i].first.c_str();
    *ms = g_last_layers[i].second;
  });
}

int hg_last_exec_node_ms(hg_ctx* ctx, double* ms_by_op) {
  return guard([&] {
    for (int i = 0; i < 11; ++i) ms_by_op[i] = ctx->last_node_ms[i];
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Client side on the GPU (hg_client.cu): secret key, encrypt_tensor, decrypt,
// decrypt_tensor (henet/graph.hpp:68-103, henet/ckks.hpp:229-263).
// ---------------------------------------------------------------------------
namespace {
using namespace hg;

// little-endian multi-word helpers for the CRT tables
void mw_mul_small(std::vector<u64>& x, u64 m) {
  unsigned __int128 carry = 0;
  for (auto& w : x) {
    const unsigned __int128 t = static_cast<unsigned __int128>(w) * m + carry;
    w = static_cast<u64>(t);
    carry = t >> 64;
  }
  if (carry) x.push_back(static_cast<u64>(carry));
}
void check_client_ctx(const Context& c) { (void)c; }
const void* client_basis(const Context& c) {
  return c.wide ? static_cast<const void*>(&c.basisw) : static_cast<const void*>(&c.basis);
}

// encrypt (henet/ckks.hpp:229-248) of `count` encoded top-level plaintexts [count][L][N]:
// ciphertext e draws from derive_seed(seed, e), stream 1 (encrypt_tensor's per-element
// seeds, and NonlinearityEngine's per-group seeds with seed = derive_seed(seed, layer)).
// ... into `ct_out` (count top-level ciphertexts); ciphertext e uses seed index e0 + e.
void encrypt_into(const Context& c, const hg_secret_key* sk, const void* pt, u64 count, u64 seed, u64 e0,
                  void* ct_out, cudaStream_t s) {
    const u32 L = static_cast<u32>(c.chain_len()), N = c.n;
    BufPtr err = c.alloc(count * L * static_cast<u64>(N) * c.word_bytes(), s);
    BufPtr flags = c.alloc(count * sizeof(int), s);
    cuda_check(cudaMemsetAsync(flags->ptr, 0, count * sizeof(int), s), "memset");
    EncArgs a{};
    a.ct = ct_out;
    a.err = err->ptr;
    a.pt = pt;
    a.sk = sk->s->ptr;
    a.e0 = static_cast<u32>(e0);
    a.flags = static_cast<int*>(flags->ptr);
    a.seed = seed;
    for (u32 i = 0; i < L; ++i) a.thr[i] = (0 - c.chain[i]) % c.chain[i];  // next_below threshold
    a.count = static_cast<u32>(count);
    a.level = L;
    a.N = N;
    check_launch(launch_enc_sample(a, client_basis(c), c.wide, s), "encrypt sample");
    // draws the counter-mode pass could not place (a rejection, u1 == 0): those ciphertexts
    // are regenerated by walking their streams, selected on the device by their flags;
    // HG_ENC_SERIAL=1 walks every stream (tests)
    const char* ser = getenv("HG_ENC_SERIAL");
    BufPtr dl;
    if (ser != nullptr && ser[0] == '1') {
      std::vector<u32> list(count);
      for (u64 e = 0; e < count; ++e) list[e] = static_cast<u32>(e);
      dl = c.alloc(count * 4, s);
      cuda_check(cudaMemcpyAsync(dl->ptr, list.data(), count * 4, cudaMemcpyHostToDevice, s), "h2d");
      cuda_check(cudaStreamSynchronize(s), "encrypt");  // the pageable list outlives the copy
    }
    check_launch(launch_enc_serial(a, dl ? static_cast<const u32*>(dl->ptr) : nullptr, static_cast<u32>(count),
                                   client_basis(c), c.wide, s),
                 "encrypt serial");
    static const bool fuse_on = [] {
      const char* e = getenv("HG_ENC_FUSE");
      return !(e != nullptr && e[0] == '0');
    }();
    const u32 lo = c.wide ? wide_narrow_lo(c.basisw, L) : L;
    if (c.wide && fuse_on && lo < L) {
      // limbs below 2^30: the error NTT and the combine in one kernel; the wide limbs as before
      check_launch(launch_enc_ntt_w(static_cast<int>(c.logn), static_cast<u64*>(a.ct), static_cast<u64*>(a.err),
                                    static_cast<const u64*>(a.pt), static_cast<const u64*>(a.sk), count, L, c.basisw,
                                    s),
                   "encrypt ntt");
      if (lo > 0) {
        EncArgs a2 = a;
        a2.limb_cnt = lo;
        check_launch(launch_enc_combine(a2, client_basis(c), c.wide, s), "encrypt combine");
      }
    } else {
      check_launch(c.wide ? launch_ntt_w(static_cast<int>(c.logn), static_cast<u64*>(a.err), count * L, L, false,
                                         c.basisw, s)
                          : launch_ntt(static_cast<int>(c.logn), static_cast<u32*>(a.err), count * L, L, false,
                                       c.basis, s),
                   "ntt");
      check_launch(launch_enc_combine(a, client_basis(c), c.wide, s), "encrypt combine");
    }
    // no synchronisation: err / flags are freed stream-ordered after the combine
}

}  // namespace

int hg_secret_key_upload(hg_ctx* ctx, const uint64_t* words, uint64_t n_words, hg_secret_key** out) {
  return guard([&] {
    require(ctx && words && out, "null argument");
    const Context& c = *ctx->c;
    check_client_ctx(c);
    const u64 full = c.chain_len() + (c.has_special ? 1 : 0), n = c.n;
    require(n_words == full * n, "secret key basis does not match the context");
    std::vector<u32> h(c.wide ? 0 : n_words);
    for (u64 i = 0; i < n_words; ++i) {
      require(words[i] < c.basis_mod(i / n), "residue out of range");
      if (!c.wide) h[i] = static_cast<u32>(words[i]);
    }
    auto* k = new hg_secret_key;
    k->ctx = ctx->c;
    k->s = c.alloc(n_words * c.word_bytes(), c.core->stream);
    cuda_check(cudaMemcpyAsync(k->s->ptr, c.wide ? static_cast<const void*>(words) : static_cast<const void*>(h.data()),
                               n_words * c.word_bytes(), cudaMemcpyHostToDevice, c.core->stream),
               "h2d");
    cuda_check(cudaStreamSynchronize(c.core->stream), "secret key");
    *out = k;
  });
}

void hg_secret_key_destroy(hg_secret_key* sk) { delete sk; }

int hg_encrypt_tensor(hg_ctx* ctx, const hg_secret_key* sk, const double* samples, uint32_t batch, uint64_t count,
                      uint64_t seed, int packing, hg_tensor* out, void* stream) {
  return guard([&] {
    require(ctx && sk && samples && out, "null argument");
    const Context& c = *ctx->c;
    check_client_ctx(c);
    cudaStream_t s = c.pick(stream);
    require(packing == HG_PACKING_REAL || packing == HG_PACKING_COMPLEX, "unknown packing mode");
    require(batch >= 1, "batch must be non-empty");
    require(batch <= (packing == HG_PACKING_REAL ? c.n / 2 : c.n), "batch exceeds slot capacity");
    if (packing == HG_PACKING_COMPLEX) require(batch % 2 == 0, "complex packing needs an even batch");
    require(count >= 1, "tensor must be non-empty");
    const u32 L = static_cast<u32>(c.chain_len()), N = c.n;
    // the samples go to the device as they are; batch_to_slots (henet/encoding.hpp:72-87),
    // encode_vector at the top level and default scale (encrypt_batch, henet/ckks.hpp:250-254)
    // and encrypt then run per chunk of 1024 ciphertexts (bounded scratch)
    const u32 n_slots = packing == HG_PACKING_REAL ? batch : batch / 2;
    BufPtr dsm = c.alloc(static_cast<u64>(batch) * count * sizeof(double), s);
    cuda_check(cudaMemcpyAsync(dsm->ptr, samples, static_cast<u64>(batch) * count * sizeof(double),
                               cudaMemcpyHostToDevice, s),
               "h2d");
    CtBatch o;
    o.packing = packing;
    o.scale = c.default_scale;
    ensure(c, o, count, 2, L, s);
    const u64 chunk = 1024, out_ct = 2ull * L * N * c.word_bytes();
    BufPtr ds = c.alloc(std::min<u64>(count, chunk) * n_slots * 2 * sizeof(double), s);
    const DeferredMagnitudes mags(c, count, s);
    for (u64 e0 = 0; e0 < count; e0 += chunk) {
      const u64 ne = std::min(chunk, count - e0);
      check_launch(launch_batch_to_slots(static_cast<const double*>(dsm->ptr), count, e0, static_cast<u32>(ne),
                                         n_slots, packing == HG_PACKING_COMPLEX, static_cast<double*>(ds->ptr), s),
                   "batch to slots");
      std::vector<unsigned long long> mant;
      std::vector<int> ex;
      BufPtr pt = encode_vectors_dev(c, static_cast<const double*>(ds->ptr), n_slots, ne, L, c.default_scale, s, mant,
                                     ex, &mags, e0);
      encrypt_into(c, sk, pt->ptr, ne, seed, e0, static_cast<char*>(o.buf->ptr) + e0 * out_ct, s);
    }
    mags.check(c, L, s);  // synchronises the stream
    out->b = o;
    out->b.shape = {static_cast<u32>(count)};
  });
}

namespace {
DecArgs dec_args(const Context& c, const hg_secret_key* sk, const void* ct, u64 count, u32 polys, u32 level) {
  // polys == 1: a plaintext (no secret key)
  require(polys == 1 || polys == 2 || polys == 3, "ciphertext must have 2 or 3 polynomials");
  require(level >= 1, "ciphertext level must be at least 1");
  DecArgs a{};
  a.ct = ct;
  a.sk = sk != nullptr ? sk->s->ptr : nullptr;
  a.count = static_cast<u32>(count);
  a.polys = polys;
  a.level = level;
  a.N = c.n;
  return a;
}
DecArgs dec_args(const Context& c, const hg_secret_key* sk, const CtBatch& ct) {
  return dec_args(c, sk, ct.buf->ptr, ct.count, ct.polys, ct.level);
}

// decode_slots(decrypt(ct)) (henet/encoding.hpp:223-264, henet/ckks.hpp:256-268) of every
// ciphertext of `b` on the GPU: slots [count][N/2][2] doubles, bit-exact.
// `count` ciphertexts at `ct` (polys x level limbs each) -> slots [count][N/2][2] in `sl`.
void decode_into(const Context& c, const hg_secret_key* sk, const void* ct, u64 count, u32 polys, u32 level,
                 double scale, double* sl, cudaStream_t s) {
    DecArgs a = dec_args(c, sk, ct, count, polys, level);
    // CRT tables for this level (decode_slots, henet/encoding.hpp:226-243)
    const u32 L = level;
    std::vector<u64> big{1};
    for (u32 i = 0; i < L; ++i) mw_mul_small(big, c.chain[i]);
    require(big.size() <= static_cast<size_t>(kCrtWords) && L <= static_cast<u32>(kCrtLimbs),
            "modulus too large for the GPU decoder");
    for (u32 i = 0; i < L; ++i) {
      a.crt.q[i] = c.chain[i];
      for (u32 j = 0; j < i; ++j) a.crt.ginv[i][j] = nt::inv(c.chain[j] % c.chain[i], c.chain[i]);
    }
    a.words = static_cast<u32>(big.size());
    for (u32 k = 0; k < a.words; ++k) a.crt.big_q[k] = big[k];
    for (u32 k = 0; k < a.words; ++k) a.crt.q_half[k] = (big[k] >> 1) | (k + 1 < a.words ? (big[k + 1] << 63) : 0);
    a.crt.fastk = 0;
    static const bool fast_on = [] {
      const char* e = getenv("HG_CRT_FAST");
      return !(e != nullptr && e[0] == '0');
    }();
    if (fast_on) {
      // the fewest leading limbs whose product exceeds 2^66 (wide c4/c5b: 2; the 30/24-bit
      // chains: 3), as long as it stays below 2^127 and leaves limbs to check
      nt::u128 qk = 1;
      u32 K = 0;
      while (K < L && K < 3 && (qk >> 66) == 0) {
        qk *= c.chain[K];
        ++K;
      }
      if ((qk >> 66) != 0 && (qk >> 126) == 0 && K < L) {
        a.crt.fastk = K;
        a.crt.q01_lo = static_cast<u64>(qk);
        a.crt.q01_hi = static_cast<u64>(qk >> 64);
        for (u32 i = 0; i < L; ++i) {
          a.crt.q01_mod[i] = static_cast<u64>(qk % c.chain[i]);
          a.crt.t64[i] = static_cast<u64>((static_cast<nt::u128>(1) << 64) % c.chain[i]);
        }
      }
    }
    {
      // 1.0L / (long double)scale (decode_slots, henet/encoding.hpp:248), x87 on the host
      const long double li = 1.0L / static_cast<long double>(scale);
      int ex = 0;
      const long double fr = std::frexp(li, &ex);  // li = fr * 2^ex, fr in [0.5, 1)
      a.inv_mant = static_cast<u64>(std::ldexp(fr, 64));
      a.inv_exp = ex - 64;
    }
    const u64 N = c.n;
    BufPtr m = c.alloc(count * L * N * c.word_bytes(), s);
    BufPtr co = c.alloc(count * N * sizeof(double), s);
    BufPtr scratch = c.alloc(count * N * sizeof(double2), s);
    a.m = m->ptr;
    a.coeffs = static_cast<double*>(co->ptr);
    const double2* roots = static_cast<const double2*>(c.fft_tables->ptr);
    check_launch(launch_dec(a, static_cast<int>(c.logn), client_basis(c), c.wide, roots, roots + N / 2,
                            static_cast<double2*>(scratch->ptr), sl, s),
                 "decrypt");
}

BufPtr decode_slots_dev(const Context& c, const hg_secret_key* sk, const CtBatch& b, cudaStream_t s) {
    BufPtr sl = c.alloc(b.count * static_cast<u64>(c.n) * sizeof(double), s);  // [count][N/2][2]
    decode_into(c, sk, b.buf->ptr, b.count, b.polys, b.level, b.scale, static_cast<double*>(sl->ptr), s);
    return sl;
}
}  // namespace

int hg_decrypt(hg_ctx* ctx, const hg_secret_key* sk, const hg_tensor* ct, uint64_t* pt_words, void* stream) {
  return guard([&] {
    require(ctx && sk && ct && pt_words, "null argument");
    const Context& c = *ctx->c;
    check_client_ctx(c);
    cudaStream_t s = c.pick(stream);
    DecArgs a = dec_args(c, sk, ct->b);
    const u64 nw = ct->b.count * ct->b.level * static_cast<u64>(c.n);
    BufPtr m = c.alloc(nw * c.word_bytes(), s);
    a.m = m->ptr;
    check_launch(launch_dec(a, static_cast<int>(c.logn), client_basis(c), c.wide, nullptr, nullptr, nullptr, nullptr, s),
                 "decrypt");
    if (c.wide) {
      cuda_check(cudaMemcpyAsync(pt_words, m->ptr, nw * 8, cudaMemcpyDeviceToHost, s), "d2h");
      cuda_check(cudaStreamSynchronize(s), "decrypt");
    } else {
      std::vector<u32> h(nw);
      cuda_check(cudaMemcpyAsync(h.data(), m->ptr, nw * 4, cudaMemcpyDeviceToHost, s), "d2h");
      cuda_check(cudaStreamSynchronize(s), "decrypt");
      for (u64 i = 0; i < nw; ++i) pt_words[i] = h[i];
    }
  });
}

int hg_decrypt_tensor(hg_ctx* ctx, const hg_secret_key* sk, const hg_tensor* ct, uint32_t batch, double* out,
                      void* stream) {
  return guard([&] {
    require(ctx && sk && ct && out, "null argument");
    const Context& c = *ctx->c;
    check_client_ctx(c);
    cudaStream_t s = c.pick(stream);
    const CtBatch& b = ct->b;
    const u32 half = c.n / 2;
    if (b.packing == HG_PACKING_REAL) {
      require(batch <= half, "batch larger than decoded slots");
    } else {
      require(batch % 2 == 0, "complex batch size must be even");
      require(batch / 2 <= half, "batch larger than decoded slots");
    }
    const u64 count = b.count, N = c.n;
    BufPtr sl = decode_slots_dev(c, sk, b, s);
    std::vector<double> h(count * N);
    cuda_check(cudaMemcpyAsync(h.data(), sl->ptr, count * N * sizeof(double), cudaMemcpyDeviceToHost, s), "d2h");
    cuda_check(cudaStreamSynchronize(s), "decrypt");
    // slots_to_batch (henet/encoding.hpp:89-107), samples[s][e]
    for (u64 e = 0; e < count; ++e) {
      const double* v = &h[e * N];
      if (b.packing == HG_PACKING_REAL) {
        for (u32 j = 0; j < batch; ++j) out[j * count + e] = v[2 * j];
      } else {
        const u32 k = batch / 2;
        for (u32 j = 0; j < k; ++j) {
          out[j * count + e] = v[2 * j];
          out[(j + k) * count + e] = v[2 * j + 1];
        }
      }
    }
  });
}

// ---------------------------------------------------------------------------
// NonlinearityEngine (henet/graph.hpp:699-741) on the GPU: decrypt + decode, ReLU or
// window max per slot, encode_vector at the top level, encrypt with
// derive_seed(derive_seed(seed, layer_seq), group) -- a drop-in hg_nonlin_fn.
// ---------------------------------------------------------------------------
struct hg_refresh_engine {
  std::shared_ptr<hg::Context> ctx;
  const hg_secret_key* sk;
  hg_secret_key sk_copy;
  uint64_t seed;
  double relu_clip = 0.0;  // > 0: ReLU refreshes clamp to [0, relu_clip] (ReLU6, BASELINE c4)
};

namespace {
u64 derive_seed_host(u64 seed, u64 tag) {  // henet/rng.hpp:101-106
  u64 z = seed + 0x9e3779b97f4a7c15ULL * (tag + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
}  // namespace

int hg_refresh_engine_create(hg_ctx* ctx, const hg_secret_key* sk, uint64_t seed, hg_refresh_engine** out) {
  return guard([&] {
    require(ctx && sk && out, "null argument");
    check_client_ctx(*ctx->c);
    auto* e = new hg_refresh_engine;
    e->ctx = ctx->c;
    e->sk_copy.ctx = sk->ctx;
    e->sk_copy.s = sk->s;  // shares the device key
    e->sk = &e->sk_copy;
    e->seed = seed;
    *out = e;
  });
}

void hg_refresh_engine_destroy(hg_refresh_engine* e) { delete e; }

int hg_refresh_engine_apply(void* engine, int kind, uint32_t window, uint32_t layer_seq, const hg_tensor* request,
                            hg_tensor* response) {
  return guard([&] {
    require(engine && request && response, "null argument");
    auto* eng = static_cast<hg_refresh_engine*>(engine);
    const Context& c = *eng->ctx;
    cudaStream_t s = c.core->stream;
    const CtBatch& b = request->b;
    require(window >= 1, "window must be at least 1");
    require(b.count % window == 0, "ciphertext count is not a multiple of the window");
    require(kind == HG_NONLIN_RELU || kind == HG_NONLIN_MAXPOOL, "unknown nonlinearity");
    if (kind == HG_NONLIN_RELU) require(window == 1, "ReLU is element-wise");
    const u64 groups = b.count / window;
    const u32 half = c.n / 2;
    const u32 L = static_cast<u32>(c.chain_len());
    using clk = std::chrono::steady_clock;
    const auto t_in = clk::now();
    // the response buffer the executor already allocated (eval_nonlinear) is reused when it
    // is large enough: one fewer layer-sized allocation at the block's memory peak
    CtBatch o;
    o.buf = std::move(response->b.buf);
    o.packing = b.packing;
    o.scale = c.default_scale;
    ensure(c, o, groups, 2, L, s);
    // in chunks of ~1024 request ciphertexts: the decode / encode / encrypt scratch is
    // ~5 words per residue, so a whole layer at once would need several times its size
    const u64 cg = std::max<u64>(1, 1024 / window);
    const u64 in_ct = static_cast<u64>(b.polys) * b.level * c.n * c.word_bytes();  // bytes per ciphertext
    const u64 out_ct = 2ull * L * c.n * c.word_bytes();
    BufPtr sl = c.alloc(std::min(groups, cg) * window * half * 2 * sizeof(double), s);
    BufPtr res = c.alloc(std::min(groups, cg) * half * 2 * sizeof(double), s);
    const u64 seed = derive_seed_host(eng->seed, layer_seq);
    const DeferredMagnitudes mags(c, groups, s);
    // HG_REFRESH_TRACE: host time of each chunk's enqueue and of the final read-back (stderr)
    static const bool trace = getenv("HG_REFRESH_TRACE") != nullptr;
    const auto t0 = clk::now();
    std::string tr;
    for (u64 g0 = 0; g0 < groups; g0 += cg) {
      const auto tc = clk::now();
      const u64 ng = std::min(cg, groups - g0);
      decode_into(c, eng->sk, static_cast<const char*>(b.buf->ptr) + g0 * window * in_ct, ng * window, b.polys,
                  b.level, b.scale, static_cast<double*>(sl->ptr), s);
      check_launch(launch_refresh_slots(static_cast<const double*>(sl->ptr), static_cast<double*>(res->ptr),
                                        static_cast<u32>(ng), window, half, kind, eng->relu_clip, s),
                   "refresh slots");
      std::vector<unsigned long long> mant;
      std::vector<int> ex;
      BufPtr pt = encode_vectors_dev(c, static_cast<const double*>(res->ptr), half, ng, L, c.default_scale, s, mant,
                                     ex, &mags, g0);
      encrypt_into(c, eng->sk, pt->ptr, ng, seed, g0, static_cast<char*>(o.buf->ptr) + g0 * out_ct, s);
      if (trace) tr += " " + std::to_string(std::chrono::duration<double, std::milli>(clk::now() - tc).count());
    }
    const auto t1 = clk::now();
    mags.check(c, L, s);  // one read-back per layer; synchronises the stream
    if (trace)
      std::fprintf(stderr, "refresh layer %u: setup %.2f ms; enqueue chunks [ms]%s; enqueue total %.2f ms, read-back wait %.2f ms\n",
                   layer_seq, std::chrono::duration<double, std::milli>(t0 - t_in).count(), tr.c_str(),
                   std::chrono::duration<double, std::milli>(t1 - t0).count(),
                   std::chrono::duration<double, std::milli>(clk::now() - t1).count());
    response->b = o;
    response->b.shape = {static_cast<u32>(groups)};
  });
}

// ---------------------------------------------------------------------------
// Wire format: put_tensor / get_tensor (henet/protocol.hpp:335-358)
// around serialize_ciphertext / deserialize_ciphertext (henet/serialize.hpp:95-124).
// Deserialisation parses the headers on the host and packs the residue words straight
// from the message into the device layout (the upload path of hg_tensor_upload, one
// segment per ciphertext), so a received request never becomes a host CipherTensor.
// ---------------------------------------------------------------------------
static_assert(__BYTE_ORDER__ == __ORDER_LITTLE_ENDIAN__, "the wire words are little-endian u64");

namespace {
struct WireReader {  // ByteReader, henet/common.hpp:90-122
  const uint8_t* d;
  u64 n, pos = 0;
  const uint8_t* take(u64 k) {
    if (k > n - pos) throw Error(HG_ERR_VALIDATION, "serialized data truncated");  // pos <= n always
    const uint8_t* p = d + pos;
    pos += k;
    return p;
  }
  uint8_t u8v() { return take(1)[0]; }
  u32 u32v() {
    const uint8_t* p = take(4);
    return static_cast<u32>(p[0]) | static_cast<u32>(p[1]) << 8 | static_cast<u32>(p[2]) << 16 |
           static_cast<u32>(p[3]) << 24;
  }
  u64 u64v() {
    const uint8_t* p = take(8);
    u64 v = 0;
    for (int i = 7; i >= 0; --i) v = (v << 8) | p[i];
    return v;
  }
};
constexpr u64 kWireHeader = 20;  // magic 4 | version 1 | N 4 | level 1 | packing 1 | scale 8 | polys 1
void put_le(uint8_t*& o, u64 v, int bytes) {
  for (int i = 0; i < bytes; ++i) *o++ = static_cast<uint8_t>(v >> (8 * i));
}
}  // namespace

int hg_tensor_deserialize(hg_ctx* ctx, const uint8_t* bytes, uint64_t len, uint64_t* consumed, hg_tensor** out,
                          void* stream) {
  return guard([&] {
    require(ctx && bytes && out, "null argument");
    const Context& c = *ctx->c;
    cudaStream_t s = c.pick(stream);
    WireReader in{bytes, len};
    std::vector<u32> dims(in.u8v());
    for (auto& d : dims) d = in.u32v();
    const u32 count = in.u32v();
    u64 elems = 1;
    for (u32 d : dims) elems *= d;
    require(count == elems, "tensor element count mismatch");
    require(count >= 1, "tensor must be non-empty");
    std::vector<const uint8_t*> segs(count);
    u32 level = 0, polys = 0;
    int packing = 0;
    double scale = 0;
    for (u32 e = 0; e < count; ++e) {
      const u64 ct_len = in.u64v();
      WireReader r{in.take(ct_len), ct_len};
      if (std::memcmp(r.take(4), "NGH2", 4) != 0) throw Error(HG_ERR_VALIDATION, "bad magic");
      if (r.u8v() != 1) throw Error(HG_ERR_VALIDATION, "unsupported wire version");
      const u32 degree = r.u32v();
      const u32 lv = r.u8v();
      const u32 pk = r.u8v();
      const u64 sbits = r.u64v();
      double sc;
      std::memcpy(&sc, &sbits, 8);
      const u32 pc = r.u8v();
      std::vector<u64> moduli(lv);
      for (auto& q : moduli) q = r.u64v();
      // check_moduli_prefix + deserialize_ciphertext's checks, in the reference's order
      require(degree == c.n, "degree does not match the context");
      require(lv >= 1 && lv <= c.chain_len(), "level outside the context chain");
      for (u32 i = 0; i < lv; ++i) require(moduli[i] == c.chain[i], "modulus list does not match the context");
      require(pc == 2 || pc == 3, "ciphertext must have 2 or 3 polynomials");
      require(pk <= 1, "unknown packing mode");
      require(sc > 0.0, "scale must be positive");
      segs[e] = r.take(static_cast<u64>(pc) * lv * c.n * 8);
      if (e == 0) {
        level = lv;
        polys = pc;
        packing = static_cast<int>(pk);
        scale = sc;
      } else if (lv != level || pc != polys || static_cast<int>(pk) != packing || sc != scale) {
        throw Error(HG_ERR_UNSUPPORTED, "device tensors carry one level, size, packing and scale for all elements");
      }
    }
    auto* t = new hg_tensor;
    std::unique_ptr<hg_tensor> guard_t(t);
    t->ctx = ctx->c;
    t->b.scale = scale;
    t->b.packing = packing;
    ensure(c, t->b, count, polys, level, s);
    t->b.shape = dims;
    const u64 seg_words = static_cast<u64>(polys) * level * c.n;
    if (!c.wide && host_narrow_enabled()) {
      require(host_narrow_upload(c.core->device, nullptr, t->b.data(), seg_words * count, level, c.n,
                                 c.chain.data(), s, segs.data(), seg_words),
              "residue out of range");
    } else {
      std::vector<u64> w(seg_words * count);
      for (u32 e = 0; e < count; ++e) std::memcpy(&w[e * seg_words], segs[e], seg_words * 8);
      const int rc = hg_tensor_upload(t, w.data(), stream);
      if (rc != HG_OK) throw Error(rc, g_last_error);
    }
    if (consumed) *consumed = in.pos;
    *out = guard_t.release();
  });
}

uint64_t hg_tensor_serialized_size(const hg_tensor* t) {
  if (!t) return 0;
  const u64 ct = kWireHeader + 8ull * t->b.level + 8ull * t->b.polys * t->b.level * t->ctx->n;
  return 1 + 4ull * t->b.shape.size() + 4 + t->b.count * (8 + ct);
}

int hg_tensor_serialize(const hg_tensor* t, uint8_t* out, uint64_t cap, void* stream) {
  return guard([&] {
    require(t && out, "null argument");
    const Context& c = *t->ctx;
    require(cap >= hg_tensor_serialized_size(t), "output buffer too small");
    const CtBatch& b = t->b;
    u64 elems = 1;
    for (u32 d : b.shape) elems *= d;
    require(elems == b.count, "tensor element count mismatch");
    const u64 seg_words = static_cast<u64>(b.polys) * b.level * c.n;
    std::vector<u64> w(seg_words * b.count);
    const int rc = hg_tensor_download(t, w.data(), stream);
    if (rc != HG_OK) throw Error(rc, g_last_error);
    uint8_t* o = out;
    put_le(o, b.shape.size(), 1);
    for (u32 d : b.shape) put_le(o, d, 4);
    put_le(o, b.count, 4);
    const u64 ct_len = kWireHeader + 8ull * b.level + 8 * seg_words;
    u64 sbits;
    std::memcpy(&sbits, &b.scale, 8);
    for (u64 e = 0; e < b.count; ++e) {
      put_le(o, ct_len, 8);
      std::memcpy(o, "NGH2", 4);
      o += 4;
      put_le(o, 1, 1);
      put_le(o, c.n, 4);
      put_le(o, b.level, 1);
      put_le(o, static_cast<u64>(b.packing), 1);
      put_le(o, sbits, 8);
      put_le(o, b.polys, 1);
      for (u32 i = 0; i < b.level; ++i) put_le(o, c.chain[i], 8);
      std::memcpy(o, &w[e * seg_words], seg_words * 8);
      o += seg_words * 8;
    }
  });
}

int hg_refresh_engine_set_relu_clip(hg_refresh_engine* e, double hi) {
  return guard([&] {
    require(e != nullptr, "null argument");
    e->relu_clip = hi;
  });
}

int hg_model_keep_encodings(hg_model* m, int on) {
  return guard([&] {
    require(m != nullptr, "null argument");
    std::lock_guard<std::mutex> g(*m->m.mu);
    m->m.keep_encodings = on != 0;
    if (!on)
      for (auto& kv : m->m.weights) kv.second.enc.clear();
  });
}

int hg_decode_vector(hg_ctx* ctx, const uint64_t* pt_words, uint64_t count, uint32_t level, double scale,
                     double* out_re_im) {
  return guard([&] {
    require(ctx && pt_words && out_re_im, "null argument");
    const Context& c = *ctx->c;
    require(level >= 1 && level <= c.chain_len(), "plaintext level out of range");
    cudaStream_t s = c.core->stream;
    const u64 nw = count * level * static_cast<u64>(c.n);
    for (u64 i = 0; i < nw; ++i) require(pt_words[i] < c.chain[(i / c.n) % level], "residue out of range");
    BufPtr d = c.alloc(nw * c.word_bytes(), s);
    if (c.wide) {
      cuda_check(cudaMemcpyAsync(d->ptr, pt_words, nw * 8, cudaMemcpyHostToDevice, s), "h2d");
    } else {
      std::vector<u32> h(pt_words, pt_words + nw);
      cuda_check(cudaMemcpyAsync(d->ptr, h.data(), nw * 4, cudaMemcpyHostToDevice, s), "h2d");
      cuda_check(cudaStreamSynchronize(s), "h2d");  // the host vector leaves scope
    }
    BufPtr sl = c.alloc(count * static_cast<u64>(c.n) * sizeof(double), s);
    decode_into(c, nullptr, d->ptr, count, 1, level, scale, static_cast<double*>(sl->ptr), s);
    cuda_check(cudaMemcpyAsync(out_re_im, sl->ptr, count * static_cast<u64>(c.n) * sizeof(double),
                               cudaMemcpyDeviceToHost, s),
               "d2h");
    cuda_check(cudaStreamSynchronize(s), "decode");
  });
}

// ---------------------------------------------------------------------------
// Multi-GPU: NCCL communicator on a context, block sharding and the
// all-gather of output ciphertexts for output-sharded layers (BASELINE c5b), so C/C++
// callers shard without torch.  NCCL is resolved at run time (dlopen "libnccl.so.2"): a
// process whose torch already loaded its NCCL shares that copy, and the library itself
// never needs NCCL unless a communicator is created.
// ---------------------------------------------------------------------------
#include <dlfcn.h>
#include <nccl.h>

namespace {
struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static const NcclApi api = [] {
    NcclApi a;
    // an NCCL the process already loaded (e.g. torch's bundled copy) wins; otherwise
    // $HG_NCCL_LIB, then the loader's libnccl.so.2
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (h == nullptr && getenv("HG_NCCL_LIB") != nullptr) h = dlopen(getenv("HG_NCCL_LIB"), RTLD_NOW);
    if (h == nullptr) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (h == nullptr) h = dlopen("libnccl.so", RTLD_NOW);
    if (h == nullptr) return a;
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(h, "ncclAllGather"));
    a.broadcast = reinterpret_cast<decltype(a.broadcast)>(dlsym(h, "ncclBroadcast"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
    return a;
  }();
  if (!api.get_unique_id || !api.comm_init_rank || !api.all_gather || !api.broadcast)
    throw Error(HG_ERR_UNSUPPORTED, "NCCL (libnccl.so.2) is not available in this process");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(HG_ERR_CUDA, std::string(what) + ": " + (nccl().error_string ? nccl().error_string(r) : "NCCL error"));
}

// contiguous block partition, sizes differ by <= 1 (paper_1908_04172_b200/dist.py shard)
void shard_range(u64 total, int rank, int nranks, u64* begin, u64* count) {
  const u64 base = total / static_cast<u64>(nranks), rem = total % static_cast<u64>(nranks);
  const u64 r = static_cast<u64>(rank);
  *begin = r * base + std::min<u64>(r, rem);
  *count = base + (r < rem ? 1 : 0);
}
}  // namespace

struct hg_comm {
  std::shared_ptr<hg::Context> ctx;
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  ~hg_comm() {
    if (comm) nccl().comm_destroy(comm);
  }
};

extern "C" {

int hg_shard_range(uint64_t total, int rank, int nranks, uint64_t* begin, uint64_t* count) {
  return guard([&] {
    require(nranks >= 1 && rank >= 0 && rank < nranks && begin && count, "bad shard arguments");
    shard_range(total, rank, nranks, begin, count);
  });
}

int hg_comm_unique_id(uint8_t* id) {
  return guard([&] {
    require(id != nullptr, "null argument");
    static_assert(sizeof(ncclUniqueId) == HG_COMM_ID_BYTES, "ncclUniqueId size");
    ncclUniqueId u;
    nccl_check(nccl().get_unique_id(&u), "ncclGetUniqueId");
    std::memcpy(id, &u, sizeof(u));
  });
}

int hg_comm_create(hg_ctx* ctx, const uint8_t* id, int nranks, int rank, hg_comm** out) {
  return guard([&] {
    require(ctx && id && out && nranks >= 1 && rank >= 0 && rank < nranks, "bad communicator arguments");
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    auto c = std::make_unique<hg_comm>();
    c->ctx = ctx->c;
    c->nranks = nranks;
    c->rank = rank;
    cuda_check(cudaSetDevice(ctx->c->core->device), "cudaSetDevice");
    nccl_check(nccl().comm_init_rank(&c->comm, nranks, u, rank), "ncclCommInitRank");
    *out = c.release();
  });
}

void hg_comm_destroy(hg_comm* c) { delete c; }

int hg_allgather_tensor(hg_comm* c, const hg_tensor* local, uint64_t total, hg_tensor** out, void* stream) {
  return guard([&] {
    require(c && local && out, "null argument");
    require(local->ctx == c->ctx, "tensor and communicator belong to different contexts");
    const Context& ctx = *c->ctx;
    cudaStream_t s = ctx.pick(stream);
    u64 b0 = 0, mine = 0;
    shard_range(total, c->rank, c->nranks, &b0, &mine);
    require(local->b.count == mine, "local tensor does not hold this rank's shard");
    const u64 ct_bytes = static_cast<u64>(local->b.polys) * local->b.level * ctx.n * ctx.word_bytes();
    u64 width = 0;
    for (int r = 0; r < c->nranks; ++r) {
      u64 b = 0, n = 0;
      shard_range(total, r, c->nranks, &b, &n);
      width = std::max(width, n);
    }
    auto* t = new hg_tensor;
    std::unique_ptr<hg_tensor> guard_t(t);
    t->ctx = c->ctx;
    t->b.packing = local->b.packing;
    t->b.scale = local->b.scale;
    t->b.shape = {static_cast<u32>(total)};
    t->b.count = total;
    t->b.polys = local->b.polys;
    t->b.level = local->b.level;
    t->b.buf = ctx.alloc(std::max<u64>(1, total * ct_bytes), s);
    if (width * static_cast<u64>(c->nranks) == total) {
      // equal blocks: gathered straight into place (a byte copy: residues unchanged)
      nccl_check(nccl().all_gather(local->b.buf->ptr, t->b.buf->ptr, width * ct_bytes, ncclUint8, c->comm, s),
                 "ncclAllGather");
    } else {
      // unequal blocks: padded send / receive buffers, then each rank's rows moved into place
      BufPtr send = ctx.alloc(width * ct_bytes, s);
      BufPtr recv = ctx.alloc(width * ct_bytes * c->nranks, s);
      cuda_check(cudaMemsetAsync(send->ptr, 0, width * ct_bytes, s), "memset");
      if (mine)
        cuda_check(cudaMemcpyAsync(send->ptr, local->b.buf->ptr, mine * ct_bytes, cudaMemcpyDeviceToDevice, s), "copy");
      nccl_check(nccl().all_gather(send->ptr, recv->ptr, width * ct_bytes, ncclUint8, c->comm, s), "ncclAllGather");
      for (int r = 0; r < c->nranks; ++r) {
        u64 b = 0, n = 0;
        shard_range(total, r, c->nranks, &b, &n);
        if (n)
          cuda_check(cudaMemcpyAsync(static_cast<char*>(t->b.buf->ptr) + b * ct_bytes,
                                     static_cast<char*>(recv->ptr) + static_cast<u64>(r) * width * ct_bytes,
                                     n * ct_bytes, cudaMemcpyDeviceToDevice, s),
                     "copy");
      }
    }
    *out = guard_t.release();
  });
}

int hg_broadcast_tensor(hg_comm* c, hg_tensor* t, int root, void* stream) {
  return guard([&] {
    require(c && t && root >= 0 && root < c->nranks, "bad broadcast arguments");
    require(t->ctx == c->ctx, "tensor and communicator belong to different contexts");
    const Context& ctx = *c->ctx;
    const u64 bytes = t->b.words(ctx.n) * ctx.word_bytes();
    nccl_check(nccl().broadcast(t->b.buf->ptr, t->b.buf->ptr, bytes, ncclUint8, root, c->comm, ctx.pick(stream)),
               "ncclBroadcast");
  });
}

}  // extern "C"
