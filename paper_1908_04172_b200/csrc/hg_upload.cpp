// SPDX-License-Identifier: Apache-2.0
//
// Host-narrowing upload of reference-format ciphertext words (hg_tensor_upload).
//
// The reference stores every residue as a u64 (RingElement, henet/modmath.hpp:257-296;
// wire order henet/serialize.hpp:61-63).  When every prime is < 2^32 the device keeps u32
// residues, so copying the u64 words over PCIe moves twice the bytes the device needs.
// Here host threads check each word against its limb's prime (the reference's
// "residue out of range" validation) and pack it to u32 into pinned chunks; each chunk is
// DMA'd on the worker's own stream as soon as it is packed, so packing and PCIe overlap
// and the bus carries 4 bytes per residue.
#include <cuda_runtime.h>
#include <emmintrin.h>
#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "hg_runtime.hpp"

namespace hg {

namespace {

// Persistent workers; run(fn) calls fn(w) for w in [0, size()) with the caller as w = 0.
class HostPool {
 public:
  explicit HostPool(int n) : n_(n) {
    for (int w = 1; w < n_; ++w) th_.emplace_back([this, w] { loop(w); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int size() const { return n_; }
  void run(const std::function<void(int)>& fn) {
    {
      std::lock_guard<std::mutex> g(mu_);
      job_ = &fn;
      pending_ = n_ - 1;
      ++gen_;
    }
    cv_.notify_all();
    fn(0);
    std::unique_lock<std::mutex> g(mu_);
    done_.wait(g, [this] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  void loop(int w) {
    uint64_t seen = 0;
    for (;;) {
      const std::function<void(int)>* job;
      {
        std::unique_lock<std::mutex> g(mu_);
        cv_.wait(g, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        job = job_;
      }
      (*job)(w);
      {
        std::lock_guard<std::mutex> g(mu_);
        if (--pending_ == 0) done_.notify_all();
      }
    }
  }
  int n_;
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_;
  const std::function<void(int)>* job_ = nullptr;
  uint64_t gen_ = 0;
  int pending_ = 0;
  bool stop_ = false;
};

constexpr u64 kChunkWords = 1u << 19;  // 2 MB of u32 per chunk (a multiple of every N)
constexpr int kSlots = 2;              // pinned chunks per worker (pack one while one is in flight)

struct Workers {
  std::unique_ptr<HostPool> pool;
  std::vector<cudaStream_t> streams;
  std::vector<cudaEvent_t> events;  // [worker][slot]
  std::vector<u32*> stage;          // [worker][slot] pinned
  std::vector<uint8_t*> dstage;     // [worker][slot] device staging of 24-bit-packed chunks
  cudaEvent_t start = nullptr;
  cudaStream_t direct = nullptr;    // the raw-u64 share: H2D + GPU narrowing
  cudaEvent_t raw_ev[4] = {};       // dynamic split: raw chunks in flight on `direct`
  std::mutex mu;                    // one upload at a time per device
};

int worker_count() {
  if (const char* e = getenv("HG_UPLOAD_THREADS")) return std::max(1, atoi(e));
  // all but two host threads (the caller's serving loop keeps launching kernels meanwhile)
  const unsigned hc = std::thread::hardware_concurrency();
  return static_cast<int>(std::min(16u, std::max(1u, hc > 4 ? hc - 2 : hc)));
}

Workers& workers(int device) {
  static std::mutex mu;
  static std::map<int, std::unique_ptr<Workers>> all;
  std::lock_guard<std::mutex> g(mu);
  auto& w = all[device];
  if (!w) {
    w = std::make_unique<Workers>();
    // the packers, plus one thread that only feeds raw chunks to the copy engine (it sleeps on
    // events between chunks; idle with the static split)
    const int n = worker_count() + 1;
    w->pool = std::make_unique<HostPool>(n);
    w->streams.resize(n);
    w->events.resize(static_cast<size_t>(n) * kSlots);
    w->stage.resize(static_cast<size_t>(n) * kSlots);
    // the upload's small kernels (24-bit unpack, raw-share narrowing) run at the highest stream
    // priority, so an execute already filling the SMs does not hold the next step's input back
    // (HG_UPLOAD_PRIORITY=0: default priority)
    int lo_pri = 0, hi_pri = 0;
    cudaDeviceGetStreamPriorityRange(&lo_pri, &hi_pri);
    const char* pe = getenv("HG_UPLOAD_PRIORITY");
    const int pri = (pe != nullptr && pe[0] == '0') ? 0 : hi_pri;
    for (int i = 0; i < n; ++i)
      cuda_check(cudaStreamCreateWithPriority(&w->streams[i], cudaStreamNonBlocking, pri), "stream");
    for (auto& e : w->events) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    for (auto& p : w->stage)
      cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&p), kChunkWords * 4, cudaHostAllocPortable), "pinned stage");
    w->dstage.resize(w->stage.size());
    for (auto& p : w->dstage) cuda_check(cudaMalloc(reinterpret_cast<void**>(&p), kChunkWords * 4), "device stage");
    cuda_check(cudaEventCreateWithFlags(&w->start, cudaEventDisableTiming), "event");
    cuda_check(cudaStreamCreateWithPriority(&w->direct, cudaStreamNonBlocking, pri), "stream");
    for (auto& e : w->raw_ev)
      cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming | cudaEventBlockingSync), "event");
  }
  return *w;
}

// One limb run (n words, n % 4 == 0; dst 16-byte aligned): u64 -> u32 with streaming stores
// (no read-for-ownership of the staging lines).  False if some word is >= q (q < 2^31): a
// high half is non-zero, or the low half is >= q.
inline bool pack_run(const u64* src, u32* dst, u32 n, u32 q) {
  const __m128i bias = _mm_set1_epi32(static_cast<int>(0x80000000u));
  const __m128i qb = _mm_set1_epi32(static_cast<int>((q - 1) ^ 0x80000000u));
  __m128i hi = _mm_setzero_si128(), over = _mm_setzero_si128();
  const __m128i* s = reinterpret_cast<const __m128i*>(src);
  __m128i* d = reinterpret_cast<__m128i*>(dst);
  for (u32 j = 0; j < n / 4; ++j) {
    const __m128i a = _mm_loadu_si128(s + 2 * j), c = _mm_loadu_si128(s + 2 * j + 1);
    const __m128i lo = _mm_unpacklo_epi64(_mm_shuffle_epi32(a, 0x08), _mm_shuffle_epi32(c, 0x08));
    hi = _mm_or_si128(hi, _mm_unpacklo_epi64(_mm_shuffle_epi32(a, 0x0D), _mm_shuffle_epi32(c, 0x0D)));
    over = _mm_or_si128(over, _mm_cmpgt_epi32(_mm_xor_si128(lo, bias), qb));  // lo > q - 1 (unsigned)
    _mm_stream_si128(d + j, lo);
  }
  return _mm_movemask_epi8(_mm_cmpeq_epi32(_mm_or_si128(hi, over), _mm_setzero_si128())) == 0xFFFF;
}

// AVX-512 variant (one 64-byte load, one unsigned compare against q over the whole u64 word,
// one VPMOVQD truncation and one 32-byte streaming store per 8 words); picked at run time
// when the host supports it (HG_UPLOAD_AVX512=0 keeps the SSE2 loop).
__attribute__((target("avx512f,avx512vl"))) inline bool pack_run_avx512(const u64* src, u32* dst, u32 n, u32 q) {
  const __m512i qv = _mm512_set1_epi64(static_cast<long long>(q));
  __mmask8 bad0 = 0, bad1 = 0;
  u32 j = 0;
  for (; j + 16 <= n; j += 16) {
    const __m512i a = _mm512_loadu_si512(src + j), c = _mm512_loadu_si512(src + j + 8);
    bad0 |= _mm512_cmpge_epu64_mask(a, qv);
    bad1 |= _mm512_cmpge_epu64_mask(c, qv);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + j), _mm512_cvtepi64_epi32(a));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + j + 8), _mm512_cvtepi64_epi32(c));
  }
  for (; j + 8 <= n; j += 8) {
    const __m512i a = _mm512_loadu_si512(src + j);
    bad0 |= _mm512_cmpge_epu64_mask(a, qv);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + j), _mm512_cvtepi64_epi32(a));
  }
  bool ok = (bad0 | bad1) == 0;
  if (j < n) ok = pack_run(src + j, dst + j, n - j, q) && ok;  // n % 4 == 0 tail
  return ok;
}

// 16 words -> 16 u32 lanes with each fourth byte dropped (48 valid bytes), range-checked
__attribute__((target("avx512f,avx512vl,avx512bw,avx512vbmi"))) inline __m512i pack24_x16(const u64* p, __m512i qv,
                                                                                          __m512i drop,
                                                                                          __mmask8& bad) {
  const __m512i a = _mm512_loadu_si512(p), b = _mm512_loadu_si512(p + 8);
  bad |= _mm512_cmpge_epu64_mask(a, qv) | _mm512_cmpge_epu64_mask(b, qv);
  return _mm512_permutexvar_epi8(
      drop, _mm512_inserti64x4(_mm512_castsi256_si512(_mm512_cvtepi64_epi32(a)), _mm512_cvtepi64_epi32(b), 1));
}

// 24-bit limbs (q < 2^24, five of the six c2 primes) cross the bus as 3 bytes per residue:
// per 64 words, eight 64-byte loads, eight unsigned compares against q, VPMOVQD to u32, VPERMB
// to drop each fourth byte and two-source VPERMT2B to splice the 48-byte pieces into three
// full 64-byte streaming stores.  dst 64-byte aligned, n % 64 == 0.
__attribute__((target("avx512f,avx512vl,avx512bw,avx512vbmi"))) inline bool pack24_run_avx512(const u64* src,
                                                                                               uint8_t* dst, u32 n,
                                                                                               u32 q) {
  alignas(64) static const uint8_t kDrop[64] = {0,  1,  2,  4,  5,  6,  8,  9,  10, 12, 13, 14, 16, 17, 18, 20,
                                                21, 22, 24, 25, 26, 28, 29, 30, 32, 33, 34, 36, 37, 38, 40, 41,
                                                42, 44, 45, 46, 48, 49, 50, 52, 53, 54, 56, 57, 58, 60, 61, 62,
                                                0,  0,  0,  0,  0,  0,  0,  0,  0,  0,  0,  0,  0,  0,  0,  0};
  alignas(64) static uint8_t kJ0[64], kJ1[64], kJ2[64];
  static const bool init = [] {
    for (int i = 0; i < 64; ++i) {
      kJ0[i] = static_cast<uint8_t>(i < 48 ? i : 64 + (i - 48));       // p0[0..47] ++ p1[0..15]
      kJ1[i] = static_cast<uint8_t>(i < 32 ? 16 + i : 64 + (i - 32));  // p1[16..47] ++ p2[0..31]
      kJ2[i] = static_cast<uint8_t>(i < 16 ? 32 + i : 64 + (i - 16));  // p2[32..47] ++ p3[0..47]
    }
    return true;
  }();
  (void)init;
  const __m512i drop = _mm512_load_si512(kDrop), j0 = _mm512_load_si512(kJ0), j1 = _mm512_load_si512(kJ1),
                j2 = _mm512_load_si512(kJ2);
  const __m512i qv = _mm512_set1_epi64(static_cast<long long>(q));
  __mmask8 bad = 0;
  for (u32 j = 0; j < n; j += 64) {
    const __m512i p0 = pack24_x16(src + j, qv, drop, bad), p1 = pack24_x16(src + j + 16, qv, drop, bad),
                  p2 = pack24_x16(src + j + 32, qv, drop, bad), p3 = pack24_x16(src + j + 48, qv, drop, bad);
    __m512i* d = reinterpret_cast<__m512i*>(dst + 3 * j);
    _mm512_stream_si512(d, _mm512_permutex2var_epi8(p0, j0, p1));
    _mm512_stream_si512(d + 1, _mm512_permutex2var_epi8(p1, j1, p2));
    _mm512_stream_si512(d + 2, _mm512_permutex2var_epi8(p2, j2, p3));
  }
  return bad == 0;
}

bool use_pack24() {
  static const bool on = [] {
    const char* e = getenv("HG_UPLOAD_PACK24");
    if (e != nullptr && e[0] == '0') return false;
    __builtin_cpu_init();
    return __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512vl") &&
           __builtin_cpu_supports("avx512bw") && __builtin_cpu_supports("avx512vbmi");
  }();
  return on;
}

// One block per limb run of a packed chunk: run r (global run R0 + r, limb (R0 + r) % level)
// starts after the runs before it, 3 bytes per residue for the limbs in mask24, else 4.
__global__ void k_unpack24(const uint8_t* packed, u32* dst, u32 N, u32 R0, u32 level, u32 mask24) {
  const u32 r = blockIdx.x;
  u64 off = 0;
  for (u32 j = 0; j < r; ++j) off += static_cast<u64>(N) * (((mask24 >> ((R0 + j) % level)) & 1u) ? 3 : 4);
  const bool w3 = (mask24 >> ((R0 + r) % level)) & 1u;
  u32* out = dst + static_cast<u64>(r) * N;
  if (w3) {
    const uint4* in = reinterpret_cast<const uint4*>(packed + off);  // 16 residues per 48 bytes
    for (u32 g = threadIdx.x; g < N / 16; g += blockDim.x) {
      const uint4 a = in[3 * g], b = in[3 * g + 1], c = in[3 * g + 2];
      const u32 w[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, c.x, c.y, c.z, c.w};
      u32 o[16];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const u32 b0 = w[3 * k], b1 = w[3 * k + 1], b2 = w[3 * k + 2];
        o[4 * k] = b0 & 0xFFFFFFu;
        o[4 * k + 1] = (b0 >> 24) | ((b1 & 0xFFFFu) << 8);
        o[4 * k + 2] = (b1 >> 16) | ((b2 & 0xFFu) << 16);
        o[4 * k + 3] = b2 >> 8;
      }
      uint4* d = reinterpret_cast<uint4*>(out + 16 * g);
      d[0] = make_uint4(o[0], o[1], o[2], o[3]);
      d[1] = make_uint4(o[4], o[5], o[6], o[7]);
      d[2] = make_uint4(o[8], o[9], o[10], o[11]);
      d[3] = make_uint4(o[12], o[13], o[14], o[15]);
    }
  } else {
    const uint4* in = reinterpret_cast<const uint4*>(packed + off);
    for (u32 g = threadIdx.x; g < N / 4; g += blockDim.x) reinterpret_cast<uint4*>(out)[g] = in[g];
  }
}

// Raw u64 chunk -> u32 residues with the < q check: word i of the chunk belongs to limb
// (R0 + i / N) % level (the dynamic split's raw path; the static split uses k_narrow).
struct ChainQ {
  u32 q[32];
};
__global__ void k_narrow_chunk(const ulonglong2* in, u32* out, u32 words, u32 N, u32 R0, u32 level, ChainQ cq,
                               int* bad) {
  const u32 i = (blockIdx.x * blockDim.x + threadIdx.x) * 4;  // N % 4 == 0: one limb per quad
  if (i >= words) return;
  const u32 q = cq.q[(R0 + i / N) % level];
  const ulonglong2 a = in[i / 2], b = in[i / 2 + 1];
  if (a.x >= q || a.y >= q || b.x >= q || b.y >= q) atomicExch(bad, 1);
  *reinterpret_cast<uint4*>(out + i) =
      make_uint4(static_cast<u32>(a.x), static_cast<u32>(a.y), static_cast<u32>(b.x), static_cast<u32>(b.y));
}

bool use_dynamic_split() {
  static const bool on = [] {
    const char* e = getenv("HG_UPLOAD_DYNAMIC");
    return !(e != nullptr && e[0] == '0');
  }();
  return on;
}

bool use_avx512() {
  static const bool on = [] {
    const char* e = getenv("HG_UPLOAD_AVX512");
    if (e != nullptr && e[0] == '0') return false;
    __builtin_cpu_init();
    return __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512vl");
  }();
  return on;
}

}  // namespace

std::atomic<u64> g_last_upload_h2d{0};  // hg_last_upload_h2d_bytes

double upload_direct_fraction() {
  static const double f = [] {
    const char* e = getenv("HG_UPLOAD_DIRECT_FRAC");
    const double v = e ? atof(e) : 0.15;
    return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v);
  }();
  return f;
}

bool host_narrow_enabled() {
  static const bool on = [] {
    const char* e = getenv("HG_UPLOAD_HOST_NARROW");
    return !(e != nullptr && e[0] == '0');
  }();
  return on;
}

// words: [count][polys][level][N] u64 (reference order) -> dst (device, u32, same order).
// With segs != nullptr the words come from n_words / seg_words separate, possibly unaligned
// segments (one serialized ciphertext each) instead of `words`.
// Returns false if some word is not below its limb's prime; dst is then unspecified.
bool host_narrow_upload(int device, const u64* words, u32* dst, u64 n_words, u32 level, u32 N, const u64* chain,
                        cudaStream_t s, const uint8_t* const* segs, u64 seg_words, const DirectShare* direct) {
  Workers& W = workers(device);
  std::lock_guard<std::mutex> g(W.mu);
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  // the copies are ordered after the work already queued on s (readers of dst)
  cuda_check(cudaEventRecord(W.start, s), "event");
  // Dynamic split (contiguous words with a raw share): the host packers take 2 MB chunks from
  // the front of the tensor and one feeder thread sends chunks from the back raw (u64 over the
  // bus, checked and narrowed on the GPU), a few in flight at a time, until the two meet.  How
  // much goes raw then follows the host's packing speed of the moment instead of a fixed
  // share: the packing is bound by the host's memory bandwidth, which varies from box to box
  // and from one minute to the next, while the bus has headroom.
  static const u64 max_raw_slots = [] {
    const char* e = getenv("HG_UPLOAD_RAW_SLOTS");
    return static_cast<u64>(e ? std::min(4, std::max(2, atoi(e))) : 2);  // 2: 6.80-6.88 ms per c2 upload step, 4: 6.84-6.99
  }();
  const int raw_slots = (direct != nullptr && direct->words != 0)
                            ? static_cast<int>(std::min<u64>(max_raw_slots, direct->words / kChunkWords)) : 0;
  const bool dynamic = use_dynamic_split() && segs == nullptr && raw_slots >= 2 && level <= 32 && N % 4 == 0 &&
                       W.pool->size() >= 2;
  if (dynamic) n_words += direct->words;  // the whole tensor is shared out chunk by chunk
  if (!dynamic && direct != nullptr && direct->words != 0) {
    // the raw share (words [n_words, n_words + direct->words)) crosses the bus as u64 and is
    // validated and narrowed on the GPU, alongside the host-packed chunks
    cuda_check(cudaStreamWaitEvent(W.direct, W.start, 0), "wait");
    cuda_check(cudaMemsetAsync(direct->bad, 0, sizeof(int), W.direct), "memset");
    cuda_check(cudaMemcpyAsync(direct->stage, words + n_words, direct->words * 8, cudaMemcpyHostToDevice, W.direct),
               "h2d");
    if (launch_narrow(direct->stage, dst + n_words, direct->words, level, N, *direct->basis, direct->bad, W.direct) < 0)
      throw Error(HG_ERR_CUDA, "narrow launch failed");
  }
  const int nw = W.pool->size() - 1;  // packers: workers [0, nw); worker nw is the raw feeder
  const bool avx512 = use_avx512();
  u32 mask24 = 0;  // limbs whose residues cross the bus as 3 bytes
  for (u32 l = 0; l < level && l < 32; ++l)
    if (chain[l] < (1ull << 24)) mask24 |= 1u << l;
  const bool pack24 = mask24 != 0 && level <= 32 && N % 64 == 0 && use_pack24();
  const u64 chunks = (n_words + kChunkWords - 1) / kChunkWords;
  std::atomic<bool> bad{false};
  std::atomic<int> err{0};
  std::atomic<u64> h2d{(!dynamic && direct != nullptr) ? direct->words * 8 : 0};
  std::string err_msg;
  std::mutex err_mu;
  // unclaimed chunks [lo, hi): packers claim lo, the raw feeder claims hi - 1
  std::atomic<u64> range{chunks};  // lo in the high 32 bits, hi in the low 32
  auto claim = [&](bool front, u64& c) {
    u64 r = range.load(std::memory_order_relaxed);
    for (;;) {
      const u64 lo = r >> 32, hi = r & 0xFFFFFFFFull;
      if (lo >= hi) return false;
      const u64 nr = front ? (((lo + 1) << 32) | hi) : ((lo << 32) | (hi - 1));
      if (range.compare_exchange_weak(r, nr, std::memory_order_relaxed)) {
        c = front ? lo : hi - 1;
        return true;
      }
    }
  };
  ChainQ cq{};
  for (u32 l = 0; l < level && l < 32; ++l) cq.q[l] = static_cast<u32>(chain[l]);
  W.pool->run([&](int w) {
    try {
      if (w == nw && !dynamic) return;
      cudaSetDevice(device);
      if (w == nw) {
        // raw chunks from the back, raw_slots of them in flight on the direct stream
        cuda_check(cudaStreamWaitEvent(W.direct, W.start, 0), "wait");
        cuda_check(cudaMemsetAsync(direct->bad, 0, sizeof(int), W.direct), "memset");
        u64 c = 0;
        for (int k = 0; claim(false, c); ++k) {
          const int slot = k % raw_slots;
          if (k >= raw_slots) cuda_check(cudaEventSynchronize(W.raw_ev[slot]), "event");
          const u64 b = c * kChunkWords, e = std::min(n_words, b + kChunkWords);
          u64* st = direct->stage + static_cast<u64>(slot) * kChunkWords;
          cuda_check(cudaMemcpyAsync(st, words + b, (e - b) * 8, cudaMemcpyHostToDevice, W.direct), "h2d");
          k_narrow_chunk<<<static_cast<u32>((e - b + 1023) / 1024), 256, 0, W.direct>>>(
              reinterpret_cast<const ulonglong2*>(st), dst + b, static_cast<u32>(e - b), N, static_cast<u32>(b / N),
              level, cq, direct->bad);
          cuda_check(cudaGetLastError(), "narrow chunk");
          cuda_check(cudaEventRecord(W.raw_ev[slot], W.direct), "event");
          h2d += (e - b) * 8;
        }
        return;  // the caller reads the flag back and synchronises the direct stream
      }
      cudaStream_t ws = W.streams[w];
      cuda_check(cudaStreamWaitEvent(ws, W.start, 0), "wait");
      bool my_bad = false;
      int used = 0;
      u64 c = static_cast<u64>(w);
      for (; dynamic ? claim(true, c) : c < chunks; c += dynamic ? 0 : static_cast<u64>(nw), ++used) {
        const int slot = used % kSlots;
        const size_t ei = static_cast<size_t>(w) * kSlots + slot;
        if (used >= kSlots) cuda_check(cudaEventSynchronize(W.events[ei]), "event");
        u32* out = W.stage[ei];
        const u64 b = c * kChunkWords, e = std::min(n_words, b + kChunkWords);
        u64 pbytes = 0;  // packed bytes of the chunk (pack24)
        for (u64 r = b; r < e; r += N) {  // one limb run of N words: a single prime
          // source run: contiguous words, or word (r % seg_words) of segment r / seg_words
          const u64* src = segs == nullptr
                               ? words + r
                               : reinterpret_cast<const u64*>(segs[r / seg_words] + (r % seg_words) * 8);
          const u32 q = static_cast<u32>(chain[(r / N) % level]);
          if (pack24) {
            uint8_t* ob = reinterpret_cast<uint8_t*>(out) + pbytes;
            if (q < (1u << 24)) {
              my_bad |= !pack24_run_avx512(src, ob, N, q);
              pbytes += static_cast<u64>(N) * 3;
            } else {
              my_bad |= !pack_run_avx512(src, reinterpret_cast<u32*>(ob), N, q);
              pbytes += static_cast<u64>(N) * 4;
            }
          } else {
            my_bad |= avx512 ? !pack_run_avx512(src, out + (r - b), N, q) : !pack_run(src, out + (r - b), N, q);
          }
        }
        _mm_sfence();  // the streaming stores are visible before the DMA reads the chunk
        h2d += pack24 ? pbytes : (e - b) * 4;
        if (pack24) {
          // 3-byte residues over the bus, widened to u32 on the device (k_unpack24)
          cuda_check(cudaMemcpyAsync(W.dstage[ei], out, pbytes, cudaMemcpyHostToDevice, ws), "h2d");
          k_unpack24<<<static_cast<u32>((e - b) / N), 256, 0, ws>>>(W.dstage[ei], dst + b, N, static_cast<u32>(b / N),
                                                                   level, mask24);
          cuda_check(cudaGetLastError(), "unpack24");
        } else {
          cuda_check(cudaMemcpyAsync(dst + b, out, (e - b) * 4, cudaMemcpyHostToDevice, ws), "h2d");
        }
        cuda_check(cudaEventRecord(W.events[ei], ws), "event");
      }
      if (my_bad) bad = true;
      cuda_check(cudaStreamSynchronize(ws), "upload");
    } catch (const std::exception& ex) {
      std::lock_guard<std::mutex> g2(err_mu);
      if (err.exchange(1) == 0) err_msg = ex.what();
    }
  });
  if (err.load()) throw Error(HG_ERR_CUDA, err_msg);
  g_last_upload_h2d = h2d.load();
  if (direct != nullptr && direct->words != 0) {
    int hbad = 0;
    cuda_check(cudaMemcpyAsync(&hbad, direct->bad, sizeof(int), cudaMemcpyDeviceToHost, W.direct), "d2h");
    cuda_check(cudaStreamSynchronize(W.direct), "upload");
    if (hbad != 0) bad = true;
  }
  return !bad.load();
}

}  // namespace hg
