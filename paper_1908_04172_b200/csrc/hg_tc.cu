// SPDX-License-Identifier: Apache-2.0
//
// Dense modular contraction (Dot, henet/graph.hpp:905-954) on the 5th-generation
// tensor cores: tcgen05.mma.kind::i8 with byte-plane limb decomposition.
//
// For one (poly, limb) slice, Y[m][n] = sum_k W[m][k] X[k][n] mod q with
// 24- or 30-bit residues.  Split both operands into bytes, w = sum_a w_a 2^8a,
// x = sum_b x_b 2^8b; then
//     Y = sum_s D_s 2^8s (mod q),   D_s = sum_{a+b=s} W_a X_b   (u8 x u8 -> s32)
// Each D_s accumulates in its own TMEM region; <= 4 products per s and K <= 8192
// keep D_s < 2^31.  The epilogue folds sum_s D_s (2^8s mod q) in u64 (< 2^64)
// and reduces once -- the same canonical residue the IMAD kernel and the
// reference produce.
//
// CTA tile: M = 128 outputs (one UMMA M) x N = 64 coefficients, K in steps of 32.
// Operands are K-major, no swizzle (canonical 8-row x 16-byte core matrices:
// LBO = 128 B between the two K halves, SBO = 256 B between 8-row groups).
// Weights are pre-packed into that layout once per layer (k_pack_weights_tc);
// X tiles arrive by cp.async (6-deep ring) and are split into byte planes in
// shared memory by 8 producer warps; one elected thread issues one MMA per weight
// plane against all input planes stacked along N.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "hg_tc.hpp"
#include "hg_wide.cuh"

namespace hg {

#ifndef HG_TC_STAGES
#define HG_TC_STAGES 4
#endif
// L2 prefetch size hint of the producers' input loads: a CTA reads TN residues per input row,
// the neighbouring column tiles (other CTAs in flight) the rest of the row
#ifndef HG_TC_L2PF
#define HG_TC_L2PF ".L2::256B"
#endif
constexpr int kTcM = 128, kTcN = 64, kTcK = 32, kTcS = HG_TC_STAGES;
constexpr int kTcProducers = 256;                 // 8 warps split X into byte planes
constexpr int kTcThreads = kTcProducers + 32;     // + 1 warp: bulk copies + MMA issue
constexpr int kTcPlaneA = kTcM * kTcK;            // 4096 B per weight byte plane per K step
constexpr int kTcPlaneB = kTcN * kTcK;            // 2048 B per input byte plane
#ifndef HG_TC_XS
#define HG_TC_XS 6
#endif
constexpr int kTcXS = HG_TC_XS;                          // cp.async stages of input residues (8 KB each)
constexpr int kTcCols = 512;                      // TMEM columns of the wide kernel (9 x 32 used)
#ifndef HG_TC_SMALLK
#define HG_TC_SMALLK 2048
#endif
constexpr u32 kTcSmallK = HG_TC_SMALLK;           // K at or below which the N = 32 tile is used

// XW: the input residue word -- u32, or u64 when the limbs are read straight out of a wide
// (u64) tensor (the 30-bit limbs of BASELINE c4/c5b), so no narrowed copy is needed.
// weight / plane ring depth: 5 for the one-CTA-per-SM N = 64 tile (measured 4% faster on
// c5b than 4), 4 for N = 32 (two CTAs per SM must fit)
template <int TN>
constexpr int tc_stages() { return TN == 64 ? 5 : 4; }

// Staged input rows are padded (TN + 4 residues) so the producers' transposed reads of a
// k-block hit distinct banks (see the producer loop); the wide TN = 64 ring is one stage
// shallower to stay within 227 KB, the wide TN = 32 ring 3 deep so two CTAs fit per SM.
template <int TN, typename XW>
constexpr int tc_xs() { return sizeof(XW) == 8 ? (TN == 64 ? kTcXS - 1 : 3) : kTcXS; }
#ifndef HG_DEBUG_CHECKS
#define HG_DEBUG_CHECKS 0
#endif
#ifndef HG_TC_XPAD64
#define HG_TC_XPAD64 0  // u64 staging rows unpadded (c5b: 61.3 vs 64.0 ms with 4 words of padding)
#endif
#ifndef HG_TC_ROT64
#define HG_TC_ROT64 0
#endif
template <int TN, typename XW = u32>
constexpr int tc_xpitch() { return TN + (sizeof(XW) == 8 ? HG_TC_XPAD64 : 4); }

template <int TN, typename XW = u32>
struct TcSmem {
  static constexpr int kS = tc_stages<TN>();
  uint8_t a[kS][4][kTcPlaneA];  // weight planes (K-major core matrices), filled by cp.async.bulk
  uint8_t b[kS][4][TN * kTcK];  // input planes, written by the producer warps; the planes of a
                                  // stage are consecutive, i.e. one K-major (planes*TN) x 32 matrix
  uint8_t zero_a[kTcPlaneA];      // zero weight plane: initialises the upper accumulators
  XW xs[tc_xs<TN, XW>()][kTcK][tc_xpitch<TN, XW>()];  // input residues staged by cp.async (producer ring)
  unsigned long long full_a[kS], full_b[kS], empty[kS], acc_full, acc_empty;
  u32 tmem;
};
// TMEM columns: 7 diagonal accumulators of TN columns (512 for TN = 64: one CTA per SM;
// 256 for TN = 32: two CTAs per SM, one's epilogue overlapping the other's MMAs)
template <int TN>
constexpr u32 tc_cols() { return TN == 64 ? 512u : 256u; }

// tcgen05.ld .16x256b.x1: 16 TMEM lanes x 8 columns; thread t receives lane t/4 (r[0..1]) and
// lane t/4 + 8 (r[2..3]), columns 2 (t % 4) and 2 (t % 4) + 1 (the mma C-fragment layout), so
// the 4 threads of a lane hold 8 consecutive columns: 64 contiguous bytes of a u64 output row.
__device__ __forceinline__ void tmem_ld_16x256b(u32 taddr, u32 (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr));
}

__device__ __forceinline__ u32 smem_addr(const void* p) { return static_cast<u32>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ u64 umma_desc(u32 saddr) {
  // start address, LBO = 128 B, SBO = 256 B (all >> 4), version 1 (sm100), SWIZZLE_NONE
  return static_cast<u64>((saddr >> 4) & 0x3FFF) | (static_cast<u64>(128 >> 4) << 16) |
         (static_cast<u64>(256 >> 4) << 32) | (1ull << 46);
}

// core-matrix offset of element (row r, k in [0,32)) of a K-major tile
__device__ __forceinline__ u32 cm_off(u32 r, u32 k) { return (r >> 3) * 256 + (k >> 4) * 128 + (r & 7) * 16 + (k & 15); }

__device__ __forceinline__ void mbar_init(unsigned long long* b, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(b)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, u32 parity) {
#if HG_DEBUG_CHECKS
  // self-check build (compute-sanitizer is not available on this pool): a wait that never
  // completes -- a phase/arrival-count bug -- traps instead of hanging the GPU
  for (u32 i = 0;; ++i) {
    u32 done;
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_addr(b)), "r"(parity));
    if (done) return;
    if (i == (1u << 24)) {
      printf("hg debug: mbarrier wait timed out (block %d thread %d parity %u)\n", blockIdx.x, threadIdx.x, parity);
      __trap();
    }
  }
#else
  asm volatile(
      "{\n.reg .pred p;\nLAB_WAIT%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra LAB_WAIT%=;\n}\n" ::"r"(smem_addr(b)),
      "r"(parity));
#endif
}

// self-check build: the TMEM allocation lies inside the 512 columns, at lane 0
__device__ __forceinline__ void tmem_check(u32 base, u32 cols) {
#if HG_DEBUG_CHECKS
  if ((base >> 16) != 0 || (base & 0xFFFFu) + cols > 512u) {
    printf("hg debug: bad TMEM allocation %08x (%u columns)\n", base, cols);
    __trap();
  }
#else
  (void)base;
  (void)cols;
#endif
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_addr(b)));
}

// ---------------------------------------------------------------------------
// Pack encoded weight residues [level][K][Mpad] (u32) into byte planes laid out
// as UMMA K-major tiles: Wp[limb][mt][ks][plane][4096 B].
// ---------------------------------------------------------------------------
__global__ void k_pack_weights_tc(const u32* W, uint8_t* Wp, u32 K, u32 Mpad, u32 Mtiles, u32 Ksteps, u32 level) {
  const u64 total = static_cast<u64>(level) * Mtiles * Ksteps * kTcM * kTcK;
  const u64 idx = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const u32 k = idx % kTcK;
  const u32 r = (idx / kTcK) % kTcM;
  const u64 t = idx / (kTcK * kTcM);
  const u32 ks = t % Ksteps;
  const u32 mt = (t / Ksteps) % Mtiles;
  const u32 limb = t / (static_cast<u64>(Ksteps) * Mtiles);
  const u32 kk = ks * kTcK + k, m = mt * kTcM + r;
  const u32 w = (kk < K && m < Mpad) ? W[(static_cast<u64>(limb) * K + kk) * Mpad + m] : 0u;
  uint8_t* tile = Wp + (((static_cast<u64>(limb) * Mtiles + mt) * Ksteps + ks) * 4) * kTcPlaneA;
#pragma unroll
  for (int p = 0; p < 4; ++p) tile[p * kTcPlaneA + cm_off(r, k)] = static_cast<uint8_t>(w >> (8 * p));
}

// ---------------------------------------------------------------------------
// Main kernel.  grid = (Mtiles * N/TN * position chunks, 1, polys * level), 288 threads:
//   warps 0-7  producers: X(ks) -> byte planes B[ks % S]; then the epilogue
//   warp 8     lane 0: weight planes by cp.async.bulk into A[], MMA issue, commits
// Rings: full_a (tx bytes), full_b (256 producer arrivals), empty (MMA commit).
// Batched contractions (npos > 1, a 1x1 convolution) whose k steps all fit the weight ring
// keep the weights resident and walk a chunk of a.ppc positions per CTA: iteration
// it = p * KS + ks over (position, k step); after a position's last k step the MMA commit
// arrives on acc_full, the producers drain the accumulators (epilogue) and arrive on
// acc_empty before the next position's first MMA overwrites them.
// ---------------------------------------------------------------------------
// BATCH: more than one position per CTA (the epilogue runs inside the k loop); otherwise the
// single position's epilogue follows the loop, as in a plain Dot.
template <int TN, typename XW = u32, bool BATCH = false>
__global__ void __launch_bounds__(kTcThreads, TN == 64 ? 1 : 2) k_mac_dense_tc(MacDenseTcArgs a, Basis B) {
  extern __shared__ __align__(1024) uint8_t tc_raw[];
  TcSmem<TN, XW>& S = *reinterpret_cast<TcSmem<TN, XW>*>(tc_raw);
  constexpr bool kWide = sizeof(XW) == 8;
  constexpr int kS = tc_stages<TN>();
  constexpr u32 kCols = tc_cols<TN>();
  const u32 tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // M tiles fastest: the CTAs in flight share their input columns (read from HBM once, the
  // other M tiles hit L2) while each M tile's weight planes stay L2-resident across N tiles
  const u32 ntiles = a.N / TN;
  const u32 mt = blockIdx.x % a.Mtiles;
  const u32 nt = (blockIdx.x / a.Mtiles) % ntiles, pc = blockIdx.x / a.Mtiles / ntiles;
  const u32 n0 = nt * TN;
  const u32 pos0 = pc * a.ppc, NP = min(a.ppc, a.npos - pos0);  // this CTA's positions
  const u32 poly = blockIdx.z / a.level, limb = blockIdx.z % a.level;
  const DevPrime& P = B.p[limb];
  const u32 planes = a.planes[limb];  // 3 for q < 2^24, 4 otherwise
  const u32 KS = a.Ksteps;
  const bool resident = BATCH && KS <= static_cast<u32>(kS);  // all weight k steps held at once
  const u32 IT = NP * KS;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_addr(&S.tmem)),
                 "r"(kCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  if (tid == 0) {
    for (int i = 0; i < kS; ++i) {
      mbar_init(&S.full_a[i], 1);
      mbar_init(&S.full_b[i], kTcProducers / 32);  // one arrive per producer warp
      mbar_init(&S.empty[i], 1);
    }
    mbar_init(&S.acc_full, 1);
    mbar_init(&S.acc_empty, kTcProducers / 32);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  for (u32 i = tid; i < kTcPlaneA / 16; i += kTcThreads)
    reinterpret_cast<uint4*>(S.zero_a)[i] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;\n" ::);  // generic-proxy zeros -> MMA reads
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  const u32 tmem = S.tmem;
  tmem_check(tmem, kCols);

  if (warp == kTcProducers / 32) {
    // ===== weight loader + MMA issuer (one lane) =====
    if (lane == 0) {
      const uint8_t* Wt = a.Wp + ((static_cast<u64>(limb) * a.Mtiles + mt) * KS) * 4 * kTcPlaneA;
      const u32 bytes = planes * kTcPlaneA;
      auto load_a = [&](u32 j) {
        const u32 st = j % kS;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(&S.full_a[st])),
                     "r"(bytes));
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                smem_addr(&S.a[st][0][0])),
            "l"(Wt + static_cast<u64>(j) * 4 * kTcPlaneA), "r"(bytes), "r"(smem_addr(&S.full_a[st])));
      };
      if (resident) {
        for (u32 j = 0; j < KS; ++j) load_a(j);
      } else {
        for (u32 j = 0; j < kS - 1 && j < KS; ++j) load_a(j);
      }
      // One MMA per weight plane pa against all input planes at once: B = the stage's planes
      // stacked along N (planes * 64 rows), D at TMEM column pa * 64, so input plane pb lands
      // in columns (pa + pb) * 64: the diagonal accumulator D_s, s = pa + pb, with no
      // per-(pa, pb) MMA.  idesc: D s32, A/B u8, K-major, N = planes * 64, M = 128.
      const u32 idesc = (2u << 4) | (((planes * TN) >> 3) << 17) | ((kTcM >> 4) << 24);
      const u64 zd = umma_desc(smem_addr(&S.zero_a[0]));
      // (p, ks) = (it / KS, it % KS), kept incrementally
      for (u32 it = 0, p = 0, ks = 0; it < IT; ++it, ks = (ks + 1 == KS) ? 0 : ks + 1, p += (ks == 0) ? 1 : 0) {
        const u32 st = it % kS, use = it / kS;
        if (!resident) {  // NP == 1: it == ks
          const u32 j = ks + kS - 1;
          if (j < KS) {
            if (j >= kS) mbar_wait(&S.empty[j % kS], ((j / kS) - 1) & 1);
            load_a(j);
          }
        }
        const u32 ast = resident ? ks : st;
        if (!resident || p == 0) mbar_wait(&S.full_a[ast], resident ? 0u : (use & 1));
        if (BATCH && ks == 0 && p > 0) mbar_wait(&S.acc_empty, (p - 1) & 1);  // position p-1 drained
        mbar_wait(&S.full_b[st], use & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
        const u64 bd = umma_desc(smem_addr(&S.b[st][0][0]));
        if (ks == 0) {
          // columns [planes * 64, 2 * planes * 64) (diagonals s >= planes) start at zero
          asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 0;\n" ::"r"(tmem + planes * TN),
                       "l"(zd), "l"(bd), "r"(idesc));
        }
        for (u32 pa = 0; pa < planes; ++pa) {
          const u64 ad = umma_desc(smem_addr(&S.a[ast][pa][0]));
          const u32 accum = (ks > 0 || pa > 0) ? 1u : 0u;  // pa = 0 of step 0 initialises s < planes
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + pa * TN),
              "l"(ad), "l"(bd), "r"(idesc), "r"(accum));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
            smem_addr(&S.empty[st])));
        if (ks == KS - 1)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
              smem_addr(&S.acc_full)));
      }
    }
  } else {
    // ===== producers: residues -> shared memory by cp.async (XS steps in flight, no register
    // cost), then byte planes.  Warp w owns the 16-row k-block kb = w / 4 and the column
    // block TN/4 * (w % 4) of every step; it copies exactly that block, so a __syncwarp (not
    // a CTA barrier) orders the copy and the reads.  Each thread transposes the bytes of KQ
    // consecutive k of one column n (KQ = 8 for TN = 64: one 8-byte run of a K-major core
    // matrix row per plane; KQ = 4 for TN = 32: 4 bytes) and stores them with one STS per
    // plane.  Lane -> (n, k) is chosen so that the stores of a phase cover all 32 banks
    // (plane writes bank-conflict free), and each thread walks its k rows rotated by ROT so
    // the reads of a phase do too (padded pitch TN + 4); the rotation is undone in registers.
    // One elected lane arrives per warp. =====
    constexpr int XS = tc_xs<TN, XW>();
    constexpr int XP = tc_xpitch<TN, XW>();
    constexpr int KQ = TN == 64 ? 8 : 4;              // k per thread
    constexpr int CW = TN / 4;                         // columns per warp
    // ROT: rows by which odd-phase threads rotate their reads (bank offset 16 against the
    // even phase): pitch XP words (u32) or 2 XP words (u64)
    constexpr int ROT = TN == 64 ? (sizeof(XW) == 4 ? 4 : HG_TC_ROT64) : 2;
    const u64 xelem = static_cast<u64>(a.polys) * a.x_level * a.N;  // words per input element
    const u64 xstride = a.x_kstride * xelem;
    const XW* Xb = static_cast<const XW*>(kWide ? static_cast<const void*>(a.X64) : static_cast<const void*>(a.X)) +
                   pos0 * a.x_pstride * xelem + (static_cast<u64>(poly) * a.x_level + a.limb_off + limb) * a.N + n0;
    const u64 xpstep = a.x_pstride * xelem;
    const u32 kb = warp >> 2, cb = (warp & 3) * CW;
    // this thread's column and first k within the step
    u32 n_t, k_t;
    bool rot;
    if constexpr (TN == 64) {
      n_t = cb + 8 * (lane >> 4) + (lane & 7);
      k_t = 16 * kb + 8 * ((lane >> 3) & 1);
      rot = ((lane >> 3) & 1) != 0;
    } else {
      n_t = cb + (lane & 7);
      k_t = 16 * kb + 4 * (lane >> 3);
      rot = sizeof(XW) == 4 ? ((lane >> 4) & 1) != 0 : ((lane >> 3) & 1) != 0;
    }
    constexpr int kPer = 16 / sizeof(XW);              // residues per 16-byte chunk
    constexpr int kCpr = CW / kPer;                    // chunks per row of the warp's block
    u32 ip = 0, iks = 0;  // (position, k step) of the next issue(): called for it = 0, 1, 2, ...
    auto issue = [&](u32 it) {
      const u32 p = ip, ks = iks;
      if (++iks == KS) {
        iks = 0;
        ++ip;
      }
      const XW* Xp = Xb + p * xpstep;
#pragma unroll
      for (int i = 0; i < 16 * kCpr / 32; ++i) {
        const u32 c = lane + i * 32, row = 16 * kb + c / kCpr, col = cb + (c % kCpr) * kPer;
        const u32 k = ks * kTcK + row;
        const XW* src = Xp + static_cast<u64>(k < a.K ? k : 0) * xstride + col;
        asm volatile("cp.async.cg.shared.global" HG_TC_L2PF " [%0], [%1], 16, %2;\n" ::"r"(smem_addr(&S.xs[it % XS][row][col])),
                     "l"(src), "r"(k < a.K ? 16 : 0));
      }
    };
#pragma unroll 1
    for (u32 j = 0; j < XS - 1; ++j) {
      if (j < IT) issue(j);
      asm volatile("cp.async.commit_group;\n" ::);
    }
    const u32 lg = warp & 3, ch = warp >> 2;
    const u32 m = mt * kTcM + lg * 32 + lane;
    const u32 q = P.q;
    const u32* cs = a.cs[limb];  // 2^(8s) mod q (host)
    const u32 nacc = 2 * planes - 1;
    const u32 bv = (a.bias != nullptr && poly == 0 && m < a.M) ? __ldg(&a.bias[static_cast<u64>(limb) * a.Mpad + m]) : 0u;
    // ===== epilogue of position pos0 + p: warp w reads TMEM lanes 32*(w%4).., columns
    // (w/4)*TN/2 .. +TN/2 =====
    auto epilogue = [&](u32 p) {
      mbar_wait(&S.acc_full, p & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
      // two diagonals per TMEM wait; diagonal 2 planes - 1 (read when nacc is odd) is zeroed by
      // the ks == 0 MMA and never accumulated.  D_s < 2^31 and 2^(8s) mod q < 2^30: one
      // IMAD.WIDE.U32 per term, the sum of 8 stays < 2^64.
      if constexpr (kWide) {
        // u64 outputs: rows lane/4 + {0, 8, 16, 24} of the warp's quarter, column pairs, so a
        // store instruction writes 8 rows x 64 contiguous bytes (16x256b TMEM loads)
        const u32 rb = mt * kTcM + lg * 32 + (lane >> 2), cp2 = 2 * (lane & 3);
        u64 bvr[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const u32 mi = rb + 8 * i;
          bvr[i] = (a.bias != nullptr && poly == 0 && mi < a.M) ? __ldg(&a.bias[static_cast<u64>(limb) * a.Mpad + mi]) : 0u;
        }
#pragma unroll
        for (u32 cc = 0; cc < TN / 2; cc += 8) {
          const u32 col = ch * (TN / 2) + cc;
          u64 acc[4][2];
#pragma unroll
          for (int i = 0; i < 4; ++i) acc[i][0] = acc[i][1] = 0;
          for (u32 s = 0; s < nacc; s += 2) {
            u32 ra[4], rb2[4], rc[4], rd[4];
            const u32 t0 = tmem + ((lg * 32) << 16) + s * TN + col, t1 = t0 + (16u << 16);
            tmem_ld_16x256b(t0, ra);
            tmem_ld_16x256b(t1, rb2);
            tmem_ld_16x256b(t0 + TN, rc);
            tmem_ld_16x256b(t1 + TN, rd);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
            const u32 c0 = cs[s], c1 = cs[s + 1];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              acc[0][j] += static_cast<u64>(ra[j]) * c0 + static_cast<u64>(rc[j]) * c1;
              acc[1][j] += static_cast<u64>(ra[2 + j]) * c0 + static_cast<u64>(rc[2 + j]) * c1;
              acc[2][j] += static_cast<u64>(rb2[j]) * c0 + static_cast<u64>(rd[j]) * c1;
              acc[3][j] += static_cast<u64>(rb2[2 + j]) * c0 + static_cast<u64>(rd[2 + j]) * c1;
            }
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const u32 mi = rb + 8 * i;
            if (mi >= a.M) continue;
            const u64 yei = mi * a.y_mstride + (pos0 + p) * a.y_pstride;
            u64* yp = a.Y64 + ((yei * a.polys + poly) * a.y_level + a.limb_off + limb) * a.N + n0 + col + cp2;
            *reinterpret_cast<ulonglong2*>(yp) =
                make_ulonglong2(addmod(reduce64(acc[i][0], P), static_cast<u32>(bvr[i]), q),
                                addmod(reduce64(acc[i][1], P), static_cast<u32>(bvr[i]), q));
          }
        }
      } else {
        const u64 ye = m * a.y_mstride + (pos0 + p) * a.y_pstride;  // output element
#pragma unroll
        for (u32 cc = 0; cc < TN / 2; cc += 8) {
          const u32 col = ch * (TN / 2) + cc;
          u64 acc[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) acc[i] = 0;
          for (u32 s = 0; s < nacc; s += 2) {
            u32 r[8], r2[8];
            const u32 taddr = tmem + ((lg * 32) << 16) + s * TN + col;
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                         : "r"(taddr));
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                         : "=r"(r2[0]), "=r"(r2[1]), "=r"(r2[2]), "=r"(r2[3]), "=r"(r2[4]), "=r"(r2[5]), "=r"(r2[6]),
                           "=r"(r2[7])
                         : "r"(taddr + TN));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
            const u32 c0 = cs[s], c1 = cs[s + 1];
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i] += static_cast<u64>(r[i]) * c0 + static_cast<u64>(r2[i]) * c1;
          }
          if (m < a.M) {
            u32 o[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) o[i] = addmod(reduce64(acc[i], P), bv, q);
            u32* yp = a.Y + ((ye * a.polys + poly) * a.level + limb) * a.N + n0 + col;
            *reinterpret_cast<uint4*>(yp) = make_uint4(o[0], o[1], o[2], o[3]);
            *reinterpret_cast<uint4*>(yp + 4) = make_uint4(o[4], o[5], o[6], o[7]);
          }
        }
      }
      if (p + 1 < NP) {  // the accumulators are free for the next position
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.acc_empty);
      }
    };
    for (u32 it = 0, p = 0, ks = 0; it < IT; ++it, ks = (ks + 1 == KS) ? 0 : ks + 1, p += (ks == 0) ? 1 : 0) {
      const u32 st = it % kS, use = it / kS;
      asm volatile("cp.async.wait_group %0;\n" ::"n"(XS - 2));
      __syncwarp();
      u32 v[KQ];
#pragma unroll
      for (int i = 0; i < KQ; ++i) {
        const u32 r = rot ? ((i + ROT) & (KQ - 1)) : static_cast<u32>(i);
        v[i] = static_cast<u32>(S.xs[it % XS][k_t + r][n_t]);
      }
      __syncwarp();  // step it's rows are consumed before the ring slot is refilled
      if (it + XS - 1 < IT) issue(it + XS - 1);
      asm volatile("cp.async.commit_group;\n" ::);
      // undo the rotation: w[t] = residue of k_t + t
      u32 w[KQ];
#pragma unroll
      for (int t = 0; t < KQ; ++t) w[t] = rot ? v[(t - ROT) & (KQ - 1)] : v[t];
      if (it >= static_cast<u32>(kS)) mbar_wait(&S.empty[st], (use - 1) & 1);
#pragma unroll
      for (int h = 0; h < KQ / 4; ++h) {
        // 4 x 4 byte transpose (8 PRMT): plane p gets byte p of the residues k_t + 4h .. +3
        const u32 t0 = __byte_perm(w[4 * h], w[4 * h + 1], 0x5140), t1 = __byte_perm(w[4 * h], w[4 * h + 1], 0x7362);
        const u32 t2 = __byte_perm(w[4 * h + 2], w[4 * h + 3], 0x5140),
                  t3 = __byte_perm(w[4 * h + 2], w[4 * h + 3], 0x7362);
        v[4 * h + 0] = __byte_perm(t0, t2, 0x5410);
        v[4 * h + 1] = __byte_perm(t0, t2, 0x7632);
        v[4 * h + 2] = __byte_perm(t1, t3, 0x5410);
        v[4 * h + 3] = __byte_perm(t1, t3, 0x7632);
      }
#pragma unroll
      for (u32 pl = 0; pl < 4; ++pl) {
        if (pl >= planes) break;
        uint8_t* dst = &S.b[st][pl][cm_off(n_t, k_t)];
        if constexpr (KQ == 8)
          *reinterpret_cast<uint2*>(dst) = make_uint2(v[pl], v[4 + pl]);
        else
          *reinterpret_cast<u32*>(dst) = v[pl];
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::);
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.full_b[st]);
      if constexpr (BATCH) {
        if (ks == KS - 1) epilogue(p);
      }
    }
    if constexpr (!BATCH) epilogue(0);
    asm volatile("cp.async.wait_group 0;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(kCols));
  }
}

// ---------------------------------------------------------------------------
// Wide limb: q in [2^30, 2^40), u64 residues, 5 byte planes.  Same pipeline with an
// N = 32 tile: one MMA per weight plane against the 5 input planes stacked along N
// (N = 160), D at TMEM column 32 pa, diagonals s = 0..8 in columns 32 s (288 of 512).
// D_s sums at most 5 plane pairs: 5 K 255^2 < 2^31 for K <= 6605.  The epilogue folds
// sum_s D_s (2^8s mod q) in 128 bits and reduces with the reference's Barrett128.
// ---------------------------------------------------------------------------
constexpr int kTwN = 32, kTwP = 5;
constexpr int kTwPlaneB = kTwN * kTcK;  // 1024 B

struct TcSmemW {
  uint8_t a[kTcS][kTwP][kTcPlaneA];
  uint8_t b[kTcS][kTwP][kTwPlaneB];
  uint8_t zero_a[kTcPlaneA];
  u64 xs[kTcXS][kTcK][kTwN];
  unsigned long long full_a[kTcS], full_b[kTcS], empty[kTcS], acc_full, acc_empty;
  u32 tmem;
};

__global__ void k_pack_weights_tc_w(const u64* W, uint8_t* Wp, u32 K, u32 Mpad, u32 Mtiles, u32 Ksteps) {
  const u64 total = static_cast<u64>(Mtiles) * Ksteps * kTcM * kTcK;
  const u64 idx = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= total) return;
  const u32 k = idx % kTcK;
  const u32 r = (idx / kTcK) % kTcM;
  const u64 t = idx / (kTcK * kTcM);
  const u32 ks = t % Ksteps;
  const u32 mt = t / Ksteps;
  const u32 kk = ks * kTcK + k, m = mt * kTcM + r;
  const u64 w = (kk < K && m < Mpad) ? W[static_cast<u64>(kk) * Mpad + m] : 0ull;
  uint8_t* tile = Wp + ((static_cast<u64>(mt) * Ksteps + ks) * kTwP) * kTcPlaneA;
#pragma unroll
  for (int p = 0; p < kTwP; ++p) tile[p * kTcPlaneA + cm_off(r, k)] = static_cast<uint8_t>(w >> (8 * p));
}

__global__ void __launch_bounds__(kTcThreads, 1) k_mac_dense_tc_w(MacDenseTcWArgs a, DevPrimeW P) {
  extern __shared__ __align__(1024) uint8_t tcw_raw[];
  TcSmemW& S = *reinterpret_cast<TcSmemW*>(tcw_raw);
  const u32 tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // M tiles fastest (see k_mac_dense_tc), then N tiles, then position chunks
  const u32 ntiles = a.N / kTwN;
  const u32 mt = blockIdx.x % a.Mtiles;
  const u32 n0 = ((blockIdx.x / a.Mtiles) % ntiles) * kTwN, pc = blockIdx.x / a.Mtiles / ntiles;
  const u32 pos0 = pc * a.ppc, NP = min(a.ppc, a.npos - pos0);
  const u32 poly = blockIdx.z;
  const u32 KS = a.Ksteps;
  const bool resident = KS <= static_cast<u32>(kTcS);  // see k_mac_dense_tc
  const u32 IT = NP * KS;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_addr(&S.tmem)),
                 "r"(kTcCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  if (tid == 0) {
    for (int i = 0; i < kTcS; ++i) {
      mbar_init(&S.full_a[i], 1);
      mbar_init(&S.full_b[i], kTcProducers / 32);
      mbar_init(&S.empty[i], 1);
    }
    mbar_init(&S.acc_full, 1);
    mbar_init(&S.acc_empty, kTcProducers / 32);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  for (u32 i = tid; i < kTcPlaneA / 16; i += kTcThreads) reinterpret_cast<uint4*>(S.zero_a)[i] = make_uint4(0, 0, 0, 0);
  asm volatile("fence.proxy.async.shared::cta;\n" ::);
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  const u32 tmem = S.tmem;
  tmem_check(tmem, kTcCols);

  if (warp == kTcProducers / 32) {
    if (lane == 0) {
      const uint8_t* Wt = a.Wp + (static_cast<u64>(mt) * KS) * kTwP * kTcPlaneA;
      constexpr u32 bytes = kTwP * kTcPlaneA;
      auto load_a = [&](u32 j) {
        const u32 st = j % kTcS;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(&S.full_a[st])),
                     "r"(bytes));
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                smem_addr(&S.a[st][0][0])),
            "l"(Wt + static_cast<u64>(j) * kTwP * kTcPlaneA), "r"(bytes), "r"(smem_addr(&S.full_a[st])));
      };
      if (resident) {
        for (u32 j = 0; j < KS; ++j) load_a(j);
      } else {
        for (u32 j = 0; j < kTcS - 1 && j < KS; ++j) load_a(j);
      }
      constexpr u32 idesc = (2u << 4) | (((kTwP * kTwN) >> 3) << 17) | ((kTcM >> 4) << 24);
      const u64 zd = umma_desc(smem_addr(&S.zero_a[0]));
      for (u32 it = 0, p = 0, ks = 0; it < IT; ++it, ks = (ks + 1 == KS) ? 0 : ks + 1, p += (ks == 0) ? 1 : 0) {
        const u32 st = it % kTcS, use = it / kTcS;
        if (!resident) {  // NP == 1: it == ks
          const u32 j = ks + kTcS - 1;
          if (j < KS) {
            if (j >= kTcS) mbar_wait(&S.empty[j % kTcS], ((j / kTcS) - 1) & 1);
            load_a(j);
          }
        }
        const u32 ast = resident ? ks : st;
        if (!resident || p == 0) mbar_wait(&S.full_a[ast], resident ? 0u : (use & 1));
        if (ks == 0 && p > 0) mbar_wait(&S.acc_empty, (p - 1) & 1);
        mbar_wait(&S.full_b[st], use & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
        const u64 bd = umma_desc(smem_addr(&S.b[st][0][0]));
        if (ks == 0)
          asm volatile("tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, 0;\n" ::"r"(tmem + kTwP * kTwN), "l"(zd),
                       "l"(bd), "r"(idesc));
#pragma unroll
        for (u32 pa = 0; pa < kTwP; ++pa) {
          const u64 ad = umma_desc(smem_addr(&S.a[ast][pa][0]));
          const u32 accum = (ks > 0 || pa > 0) ? 1u : 0u;
          asm volatile(
              "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + pa * kTwN),
              "l"(ad), "l"(bd), "r"(idesc), "r"(accum));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
            smem_addr(&S.empty[st])));
        if (ks == KS - 1)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
              smem_addr(&S.acc_full)));
      }
    }
  } else {
    // producers: warp w owns k rows [4w, 4w+4) of every step; lane = column
    const u64 xelem = static_cast<u64>(a.polys) * a.x_level * a.N;
    const u64 xstride = a.x_kstride * xelem, xpstep = a.x_pstride * xelem;
    const u64* Xb = a.X + pos0 * xpstep + (static_cast<u64>(poly) * a.x_level + a.limb) * a.N + n0;
    const u32 r0 = warp * 4;
    u32 ip = 0, iks = 0;  // (position, k step) of the next issue(): called for it = 0, 1, 2, ...
    auto issue = [&](u32 it) {
      const u32 p = ip, ks = iks;
      if (++iks == KS) {
        iks = 0;
        ++ip;
      }
      // 4 rows x 32 residues (u64) = 64 chunks of 16 B, two per lane; rows >= K zero-fill
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const u32 c = lane + i * 32, row = r0 + (c >> 4), c2 = (c & 15) * 2;
        const u32 k = ks * kTcK + row;
        const u64* src = Xb + p * xpstep + static_cast<u64>(k < a.K ? k : 0) * xstride + c2;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_addr(&S.xs[it % kTcXS][row][c2])),
                     "l"(src), "r"(k < a.K ? 16 : 0));
      }
    };
#pragma unroll 1
    for (u32 j = 0; j < kTcXS - 1; ++j) {
      if (j < IT) issue(j);
      asm volatile("cp.async.commit_group;\n" ::);
    }
    const u32 lg = warp & 3, ch = warp >> 2;
    for (u32 it = 0, p = 0, ks = 0; it < IT; ++it, ks = (ks + 1 == KS) ? 0 : ks + 1, p += (ks == 0) ? 1 : 0) {
      const u32 st = it % kTcS, use = it / kTcS;
      asm volatile("cp.async.wait_group %0;\n" ::"n"(kTcXS - 2));
      __syncwarp();
      u64 v[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) v[i] = S.xs[it % kTcXS][r0 + i][lane];
      __syncwarp();
      if (it + kTcXS - 1 < IT) issue(it + kTcXS - 1);
      asm volatile("cp.async.commit_group;\n" ::);
      if (it >= static_cast<u32>(kTcS)) mbar_wait(&S.empty[st], (use - 1) & 1);
#pragma unroll
      for (u32 pl = 0; pl < kTwP; ++pl) {
        const u32 sh = 8 * pl;
        const u32 b4 = static_cast<u32>((v[0] >> sh) & 255) | (static_cast<u32>((v[1] >> sh) & 255) << 8) |
                       (static_cast<u32>((v[2] >> sh) & 255) << 16) | (static_cast<u32>((v[3] >> sh) & 255) << 24);
        *reinterpret_cast<u32*>(&S.b[st][pl][cm_off(lane, r0)]) = b4;
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::);
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.full_b[st]);
      if (ks != KS - 1) continue;

      // epilogue of position pos0 + p: warp w reads TMEM lanes 32 (w % 4) .., columns
      // 16 (w / 4) .. + 16, as 16x256b loads: rows lane/4 + {0, 8, 16, 24}, column pairs, so a
      // store instruction writes 8 rows x 64 contiguous bytes
      mbar_wait(&S.acc_full, p & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
      const u32 rb = mt * kTcM + lg * 32 + (lane >> 2), cp2 = 2 * (lane & 3);
#pragma unroll
      for (u32 cc = 0; cc < 16; cc += 8) {
        const u32 col = ch * 16 + cc;
        // sum_s D_s (2^(8s) mod q) with the multiplier split at bit 20: D_s < 2^31 and both
        // halves < 2^20, so each half-sum of 10 terms (diagonal 9 is zero, see k_mac_dense_tc)
        // stays < 2^55 with one IMAD.WIDE.U32 per term
        u64 al[4][2], ah[4][2];
#pragma unroll
        for (int i = 0; i < 4; ++i) al[i][0] = al[i][1] = ah[i][0] = ah[i][1] = 0;
#pragma unroll 1
        for (u32 s = 0; s < 2 * kTwP - 1; s += 2) {
          u32 ra[4], rb2[4], rc[4], rd[4];
          const u32 t0 = tmem + ((lg * 32) << 16) + s * kTwN + col, t1 = t0 + (16u << 16);
          tmem_ld_16x256b(t0, ra);
          tmem_ld_16x256b(t1, rb2);
          tmem_ld_16x256b(t0 + kTwN, rc);
          tmem_ld_16x256b(t1 + kTwN, rd);
          asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
          const u64 c = a.cs[s], c2 = a.cs[s + 1];
          const u32 cl = static_cast<u32>(c & 0xFFFFF), chh = static_cast<u32>(c >> 20);
          const u32 cl2 = static_cast<u32>(c2 & 0xFFFFF), ch2 = static_cast<u32>(c2 >> 20);
          const u32* d1[4] = {ra, ra + 2, rb2, rb2 + 2};
          const u32* d2[4] = {rc, rc + 2, rd, rd + 2};
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              al[i][j] += static_cast<u64>(d1[i][j]) * cl + static_cast<u64>(d2[i][j]) * cl2;
              ah[i][j] += static_cast<u64>(d1[i][j]) * chh + static_cast<u64>(d2[i][j]) * ch2;
            }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const u32 mi = rb + 8 * i;
          if (mi >= a.M) continue;
          const u64 bvi = (a.bias != nullptr && poly == 0) ? __ldg(&a.bias[mi]) : 0ull;
          u64 o[2];
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const u64 lo = al[i][j] + (ah[i][j] << 20);
            const u64 hi = (ah[i][j] >> 44) + (lo < al[i][j] ? 1 : 0);
            o[j] = addmod_w(barrett128(lo, hi, P), bvi, P.q);
          }
          const u64 ye = mi * a.y_mstride + (pos0 + p) * a.y_pstride;
          u64* yp = a.Y + ((ye * a.polys + poly) * a.level + a.limb) * a.N + n0 + col + cp2;
          *reinterpret_cast<ulonglong2*>(yp) = make_ulonglong2(o[0], o[1]);
        }
      }
      if (p + 1 < NP) {
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
        __syncwarp();
        if (lane == 0) mbar_arrive(&S.acc_empty);
      }
    }
    asm volatile("cp.async.wait_group 0;\n" ::);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(kTcCols));
  }
}

// ---------------------------------------------------------------------------
// int8 tensor-core peak probe (the tensor roofline denominator): one CTA per SM issues
// back-to-back M=128 x N=256 x K=32 kind::i8 MMAs from static shared-memory operands in
// this file's layout (scripts/umma_probe.cu sweeps N).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128, 1) k_umma_probe(u32 iters) {
  extern __shared__ __align__(1024) uint8_t pr_raw[];
  __shared__ u32 tmem;
  __shared__ __align__(8) unsigned long long bar;
  for (u32 i = threadIdx.x; i < (4096 + 256 * 32) / 4; i += blockDim.x)
    reinterpret_cast<u32*>(pr_raw)[i] = i * 2654435761u;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_addr(&tmem)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::);
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  if (threadIdx.x == 0) {
    constexpr u32 idesc = (2u << 4) | ((256 >> 3) << 17) | ((128 >> 4) << 24);
    const u64 ad = umma_desc(smem_addr(pr_raw)), bd = umma_desc(smem_addr(pr_raw + 4096));
    for (u32 it = 0; it < iters; ++it)
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc),
          "r"(it));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_addr(&bar)));
    mbar_wait(&bar, 0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
}

double bench_tc_i8_peak(int device) {
  cudaSetDevice(device);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  cudaFuncSetAttribute(k_umma_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  const u32 iters = 20000;
  k_umma_probe<<<sms, 128, 160 * 1024>>>(100);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    k_umma_probe<<<sms, 128, 160 * 1024>>>(iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return static_cast<double>(sms) * iters * 128.0 * 256.0 * 32.0 / (best * 1e-3);  // int8 MAC/s
}

// ---------------------------------------------------------------------------
// Launchers
// ---------------------------------------------------------------------------
// Positions per CTA of a batched contraction with resident weights (HG_TC_PPC, default 16).
static u32 tc_positions_per_cta() {
  static const u32 v = [] {
    const char* e = getenv("HG_TC_PPC");
    const int x = e ? atoi(e) : 16;
    return static_cast<u32>(x < 1 ? 1 : x);
  }();
  return v;
}

u64 tc_packed_weight_bytes(u32 K, u32 M, u32 level) {
  const u32 Mtiles = (M + kTcM - 1) / kTcM, Ksteps = (K + kTcK - 1) / kTcK;
  return static_cast<u64>(level) * Mtiles * Ksteps * 4 * kTcPlaneA;
}

int launch_pack_weights_tc(const u32* W, uint8_t* Wp, u32 K, u32 M, u32 Mpad, u32 level, cudaStream_t s) {
  const u32 Mtiles = (M + kTcM - 1) / kTcM, Ksteps = (K + kTcK - 1) / kTcK;
  const u64 total = static_cast<u64>(level) * Mtiles * Ksteps * kTcM * kTcK;
  ProfScope ps("k_pack_weights_tc", s);
  k_pack_weights_tc<<<(total + 255) / 256, 256, 0, s>>>(W, Wp, K, Mpad, Mtiles, Ksteps, level);
  return 1;
}

u64 tc_packed_weight_bytes_w(u32 K, u32 M) {
  const u32 Mtiles = (M + kTcM - 1) / kTcM, Ksteps = (K + kTcK - 1) / kTcK;
  return static_cast<u64>(Mtiles) * Ksteps * kTwP * kTcPlaneA;
}

int launch_pack_weights_tc_w(const u64* W, uint8_t* Wp, u32 K, u32 M, u32 Mpad, cudaStream_t s) {
  const u32 Mtiles = (M + kTcM - 1) / kTcM, Ksteps = (K + kTcK - 1) / kTcK;
  const u64 total = static_cast<u64>(Mtiles) * Ksteps * kTcM * kTcK;
  ProfScope ps("k_pack_weights_tc_w", s);
  k_pack_weights_tc_w<<<(total + 255) / 256, 256, 0, s>>>(W, Wp, K, Mpad, Mtiles, Ksteps);
  return 1;
}

int launch_mac_dense_tc_w(MacDenseTcWArgs a, const void* P, cudaStream_t s) {
  a.Mtiles = (a.M + kTcM - 1) / kTcM;
  a.Ksteps = (a.K + kTcK - 1) / kTcK;
  if (a.N % kTwN != 0 || a.K > 6605 || a.K == 0) return -1;  // 5 K 255^2 < 2^31
  if (a.npos == 0) a.npos = 1;
  if (a.x_kstride == 0) a.x_kstride = 1;
  if (a.y_mstride == 0) a.y_mstride = 1;
  a.ppc = a.Ksteps <= static_cast<u32>(kTcS) ? std::min(a.npos, tc_positions_per_cta()) : 1u;
  const u64 ctas = static_cast<u64>(a.Mtiles) * (a.N / kTwN) * ((a.npos + a.ppc - 1) / a.ppc);
  if (ctas >= (1ull << 31)) return -1;
  constexpr size_t smem = sizeof(TcSmemW) > 120 * 1024 ? sizeof(TcSmemW) : 120 * 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_mac_dense_tc_w, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    attr = true;
  }
  dim3 grid(static_cast<u32>(ctas), 1, a.polys);
  ProfScope ps("k_mac_dense_tc_w", s);
  k_mac_dense_tc_w<<<grid, kTcThreads, smem, s>>>(a, *static_cast<const DevPrimeW*>(P));
  return 1;
}

template <int TN, typename XW, bool BATCH>
static void tc_launch_k(const MacDenseTcArgs& a, const Basis& B, cudaStream_t s) {
  // TN = 64: request enough shared memory that only one CTA is resident per SM (512 TMEM
  // columns), so no CTA spins in tcgen05.alloc; TN = 32: two CTAs of 256 columns.
  constexpr size_t smem = TN == 64 ? (sizeof(TcSmem<TN, XW>) > 120 * 1024 ? sizeof(TcSmem<TN, XW>) : 120 * 1024)
                                   : sizeof(TcSmem<TN, XW>);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_mac_dense_tc<TN, XW, BATCH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    attr = true;
  }
  dim3 grid(a.Mtiles * (a.N / TN) * ((a.npos + a.ppc - 1) / a.ppc), 1, a.polys * a.level);
  ProfScope ps("k_mac_dense_tc", s);
  k_mac_dense_tc<TN, XW, BATCH><<<grid, kTcThreads, smem, s>>>(a, B);
}

template <int TN, typename XW>
static void tc_launch(MacDenseTcArgs a, const Basis& B, cudaStream_t s) {
  a.ppc = a.Ksteps <= static_cast<u32>(tc_stages<TN>()) ? std::min(a.npos, tc_positions_per_cta()) : 1u;
  if constexpr (TN == 32) {  // batched contractions have small K (the N = 32 tile)
    if (a.ppc > 1) {
      tc_launch_k<TN, XW, true>(a, B, s);
      return;
    }
  }
  tc_launch_k<TN, XW, false>(a, B, s);
}

int launch_mac_dense_tc(MacDenseTcArgs a, const Basis& B, cudaStream_t s) {
  a.Mtiles = (a.M + kTcM - 1) / kTcM;
  a.Ksteps = (a.K + kTcK - 1) / kTcK;
  if (a.N % 64 != 0 || a.K > 8192 || a.K == 0) return -1;
  if (a.npos == 0) a.npos = 1;
  if (a.x_kstride == 0) a.x_kstride = 1;
  if (a.y_mstride == 0) a.y_mstride = 1;
  if (static_cast<u64>(a.Mtiles) * (a.N / 32) * a.npos >= (1ull << 31)) return -1;
  for (u32 l = 0; l < a.level; ++l) {
    const u64 q = B.p[l].q;
    u64 c = 1;
    for (int i = 0; i < 7; ++i) {
      a.cs[l][i] = static_cast<u32>(c);
      c = (c << 8) % q;
    }
    a.cs[l][7] = 0;
  }
  // short contractions are dominated by per-CTA prologue/epilogue: two CTAs per SM overlap them
  static const int tn_env = [] {
    const char* e = getenv("HG_TC_N");
    return e ? atoi(e) : 0;
  }();
  const int tn = tn_env ? tn_env : (a.K <= kTcSmallK ? 32 : 64);
  const bool wio = a.X64 != nullptr;
  if (tn == 32)
    wio ? tc_launch<32, u64>(a, B, s) : tc_launch<32, u32>(a, B, s);
  else
    wio ? tc_launch<64, u64>(a, B, s) : tc_launch<64, u32>(a, B, s);
  return 1;
}

}  // namespace hg
