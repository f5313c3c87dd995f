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
  cudaEvent_t start = nullptr;
  cudaStream_t direct = nullptr;    // the raw-u64 share: H2D + GPU narrowing
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
    const int n = worker_count();
    w->pool = std::make_unique<HostPool>(n);
    w->streams.resize(n);
    w->events.resize(static_cast<size_t>(n) * kSlots);
    w->stage.resize(static_cast<size_t>(n) * kSlots);
    for (int i = 0; i < n; ++i) cuda_check(cudaStreamCreateWithFlags(&w->streams[i], cudaStreamNonBlocking), "stream");
    for (auto& e : w->events) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    for (auto& p : w->stage)
      cuda_check(cudaHostAlloc(reinterpret_cast<void**>(&p), kChunkWords * 4, cudaHostAllocPortable), "pinned stage");
    cuda_check(cudaEventCreateWithFlags(&w->start, cudaEventDisableTiming), "event");
    cuda_check(cudaStreamCreateWithFlags(&w->direct, cudaStreamNonBlocking), "stream");
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
  if (direct != nullptr && direct->words != 0) {
    // the raw share (words [n_words, n_words + direct->words)) crosses the bus as u64 and is
    // validated and narrowed on the GPU, alongside the host-packed chunks
    cuda_check(cudaStreamWaitEvent(W.direct, W.start, 0), "wait");
    cuda_check(cudaMemsetAsync(direct->bad, 0, sizeof(int), W.direct), "memset");
    cuda_check(cudaMemcpyAsync(direct->stage, words + n_words, direct->words * 8, cudaMemcpyHostToDevice, W.direct),
               "h2d");
    if (launch_narrow(direct->stage, dst + n_words, direct->words, level, N, *direct->basis, direct->bad, W.direct) < 0)
      throw Error(HG_ERR_CUDA, "narrow launch failed");
  }
  const int nw = W.pool->size();
  const bool avx512 = use_avx512();
  const u64 chunks = (n_words + kChunkWords - 1) / kChunkWords;
  std::atomic<bool> bad{false};
  std::atomic<int> err{0};
  std::string err_msg;
  std::mutex err_mu;
  W.pool->run([&](int w) {
    try {
      cudaSetDevice(device);
      cudaStream_t ws = W.streams[w];
      cuda_check(cudaStreamWaitEvent(ws, W.start, 0), "wait");
      bool my_bad = false;
      int used = 0;
      for (u64 c = static_cast<u64>(w); c < chunks; c += static_cast<u64>(nw), ++used) {
        const int slot = used % kSlots;
        const size_t ei = static_cast<size_t>(w) * kSlots + slot;
        if (used >= kSlots) cuda_check(cudaEventSynchronize(W.events[ei]), "event");
        u32* out = W.stage[ei];
        const u64 b = c * kChunkWords, e = std::min(n_words, b + kChunkWords);
        for (u64 r = b; r < e; r += N) {  // one limb run of N words: a single prime
          // source run: contiguous words, or word (r % seg_words) of segment r / seg_words
          const u64* src = segs == nullptr
                               ? words + r
                               : reinterpret_cast<const u64*>(segs[r / seg_words] + (r % seg_words) * 8);
          const u32 q = static_cast<u32>(chain[(r / N) % level]);
          my_bad |= avx512 ? !pack_run_avx512(src, out + (r - b), N, q) : !pack_run(src, out + (r - b), N, q);
        }
        _mm_sfence();  // the streaming stores are visible before the DMA reads the chunk
        cuda_check(cudaMemcpyAsync(dst + b, out, (e - b) * 4, cudaMemcpyHostToDevice, ws), "h2d");
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
  if (direct != nullptr && direct->words != 0) {
    int hbad = 0;
    cuda_check(cudaMemcpyAsync(&hbad, direct->bad, sizeof(int), cudaMemcpyDeviceToHost, W.direct), "d2h");
    cuda_check(cudaStreamSynchronize(W.direct), "upload");
    if (hbad != 0) bad = true;
  }
  return !bad.load();
}

}  // namespace hg
