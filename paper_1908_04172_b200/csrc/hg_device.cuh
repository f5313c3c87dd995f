// SPDX-License-Identifier: Apache-2.0
//
// Device-side modular arithmetic and the per-limb negacyclic NTT block.
//
// Every prime handled here is < 2^30, so residues live in u32 and Harvey's lazy
// butterflies can keep values in [0, 4q) < 2^32.  Results written to HBM are
// always canonical ([0, q)), which is what makes them bit-identical to the
// reference: the reference's outputs are canonical residues of the same
// mathematical values (henet/modmath.hpp:149-165, 338-377).
//
// NTT convention (henet/modmath.hpp:303-377): forward is Cooley-Tukey with
// twiddle root_powers[m + i] = psi^bitrev(m + i) at stage m (t = N / 2m),
// pairs (j, j + t); inverse is Gentleman-Sande with psi^-bitrev(m + i) and a
// final multiply by N^-1, which is folded into the last inverse stage here.
// The tables keep the reference's index order, so output index i holds the
// evaluation at psi^(2 bitrev(i) + 1) exactly as ntt_forward_limb does.
#pragma once

#include <cstdint>

namespace hg {

using u32 = uint32_t;
using u64 = uint64_t;
using i32 = int32_t;

#ifndef HG_MAX_PRIMES
#define HG_MAX_PRIMES 24
#endif
constexpr int kMaxPrimes = HG_MAX_PRIMES;

#ifndef HG_DEBUG_CHECKS
#define HG_DEBUG_CHECKS 0  // self-check build: mbarrier wait timeouts and TMEM allocation checks trap
#endif
#ifndef HG_NTT_TWS_MINB
#define HG_NTT_TWS_MINB 4  // ... and the kernels with staged pass-B twiddles (Ntt<LOGN, true>)
#endif
#ifndef HG_RESCALE_MINB
#define HG_RESCALE_MINB 4  // rescale: correction row in TMEM, 41 KB smem, 64 registers
#endif
#ifndef HG_RESCALE_TMEM_CELLS
#define HG_RESCALE_TMEM_CELLS 32  // rescale keeps one correction row: half the TMEM columns
#endif
#ifndef HG_DIGITS_MINB
#define HG_DIGITS_MINB 4
#endif
#ifndef HG_KEYSW_MINB
#define HG_KEYSW_MINB 4  // key switch: accumulators in TMEM (4 x 128 columns), 41 KB smem
#endif
#ifndef HG_KEYSW_PREFETCH
#define HG_KEYSW_PREFETCH 1  // next digit loaded into registers during the key products
#endif
#ifndef HG_BFLY_ALU_ADD
#define HG_BFLY_ALU_ADD 1  // butterfly sum X + T as an ALU-pipe min(X + T, ~0) (keeps ptxas from IMAD.IADD)
#endif
// Timing-only switches (results are wrong; used to attribute kernel time, never shipped)
#ifndef HG_T_NOF
#define HG_T_NOF 0
#endif
#ifndef HG_T_NOBAR
#define HG_T_NOBAR 0
#endif
#ifndef HG_T_NOXCHG
#define HG_T_NOXCHG 0
#endif
#if HG_T_NOBAR
#define HG_NTT_SYNC() ((void)0)
#else
#define HG_NTT_SYNC() __syncthreads()
#endif
#ifndef HG_MODDOWN_TOPINV
#define HG_MODDOWN_TOPINV 1  // merged rescale: the dropped limb takes one INTT, not NTT + INTT
#endif
// Mod-down: 4 CTAs per SM at 64 registers without a register prefetch of the accumulator row.
// With the dropped limb's single INTT and the P^-1 factor folded into the key the body fits 64
// registers without spills; alone it is as fast as 3 CTAs per SM (0.31 vs 0.30 ms per c2 step,
// 0.32 for the old 2 CTAs/SM + prefetch at 127 registers), and its small CTAs share SMs better
// with the other half-batch's key switch: step 1.891 -> 1.834 ms (profiles/r3_experiments.md).
#ifndef HG_MODDOWN_PREFETCH
#define HG_MODDOWN_PREFETCH 0  // 1: accumulator row loaded before the transform (registers)
#endif
#ifndef HG_MODDOWN_MINB
#define HG_MODDOWN_MINB 4
#endif
#ifndef HG_NTT14_MINB
#define HG_NTT14_MINB 2  // N = 2^14 transforms (512 threads): 2 CTAs per SM, 64 registers
#endif
#ifndef HG_NTT_MINB
#define HG_NTT_MINB 2  // CTAs per SM the NTT kernels are register-budgeted for (N <= 2^13)
#endif

// Per-basis-modulus constants.  Passed by value (kernel parameter space).
struct DevPrime {
  u32 q;
  u32 two_q;
  u32 half;      // floor(q / 2)
  u32 mu32;      // floor(2^32 / q)                -> reduce a u32 to [0, q)
  u64 mu64;      // floor(2^64 / q)                -> Barrett of a u64 accumulator
  u32 r32;       // 2^32 mod q                      -> accumulator folding
  u32 ninv;      // N^-1 mod q
  u32 ninv_sh;   // floor(ninv * 2^32 / q)
  u32 w1n;       // inv_root_powers[1] * N^-1 mod q (last inverse stage)
  u32 w1n_sh;
  u32 bsh;       // k - 1, k = bit length of q       -> product Barrett (mulmod)
  u32 bmu;       // floor(2^(k+31) / q) (< 2^32)
  u32 pad_;
  // Twiddles staged per NTT pass (see Ntt below): pass A (uniform over the CTA)
  // from the kernel parameter block, passes B / C from per-thread rows of 32
  // (value, shoup) pairs in the exact order the unrolled stages consume them.
  uint2 twA[32];       // root_powers[1..31]      (psi^bitrev(i), shoup)
  uint2 itwA[32];      // inv_root_powers[1..31]
  // Pass C: twiddle psi^bitrev(idx) = V(stage, c, g) * T_stage(tid) because idx's
  // bit fields from (c, g) and from tid are disjoint and bit reversal is additive
  // over disjoint fields.  V is uniform (here); T is one value per thread and stage.
  uint2 tvC[32];       // forward V, consumption order
  uint2 itvC[32];      // inverse V
  const uint2* fwdB;   // [2^MB rows][32] staged pass-B rows
  const uint2* fwdT;   // [T rows][2^CB]: F_k(tid) = prod_{b in bits(k)} T_b(tid) (Ntt::scale_C)
  const uint2* invB;
  const uint2* invT;
};

struct Basis {
  DevPrime p[kMaxPrimes];  // chain moduli first, special prime at index chain_len
};

// ---------------------------------------------------------------------------
// Scalar modular helpers
// ---------------------------------------------------------------------------

// x in [0, 2q) -> [0, q): unsigned min picks x - q only when it did not wrap.
__device__ __forceinline__ u32 csub(u32 x, u32 q) { return min(x, x - q); }

// Shoup multiplication by a constant w (< q) with companion wsh = floor(w 2^32 / q).
// For any x < 2^32 the result is congruent to x*w and lies in [0, 2q) (q < 2^31).
__device__ __forceinline__ u32 mul_shoup_lazy(u32 x, u32 w, u32 wsh, u32 q) {
  const u32 qhat = __umulhi(x, wsh);
  return x * w - qhat * q;
}

__device__ __forceinline__ u32 mul_shoup(u32 x, u32 w, u32 wsh, u32 q) {
  return csub(mul_shoup_lazy(x, w, wsh, q), q);
}

// Reduce any u32 into [0, q).
__device__ __forceinline__ u32 reduce32(u32 x, const DevPrime& P) {
  const u32 qhat = __umulhi(x, P.mu32);
  u32 r = x - qhat * P.q;  // < 2q
  return csub(r, P.q);
}

// Reduce any u64 into [0, q) (Barrett with mu = floor(2^64/q); remainder < 2q).
__device__ __forceinline__ u32 reduce64(u64 x, const DevPrime& P) {
  const u64 qhat = __umul64hi(x, P.mu64);
  u32 r = static_cast<u32>(x - qhat * static_cast<u64>(P.q));
  return csub(r, P.q);
}

// a * b mod q for a, b < 2^k (k = bit length of q, so any canonical residues): Barrett on
// the top k+1 bits of the product, x' = floor(ab / 2^(k-1)) < 2^(k+1),
// qhat = floor(x' * floor(2^(k+31)/q) / 2^32) in [floor(ab/q) - 2, floor(ab/q)], so the low
// word of ab - qhat*q is the remainder plus at most 2q (< 2^32 for q < 2^30).  One IMAD.HI
// instead of the 64x64 high product of reduce64.
// Lazy variant: congruent to a * b, in [0, 2q).
__device__ __forceinline__ u32 mulmod_lazy2(u32 a, u32 b, const DevPrime& P) {
  const u64 x = static_cast<u64>(a) * b;
  const u32 xs = static_cast<u32>(x >> P.bsh);
  const u32 r = static_cast<u32>(x) - __umulhi(xs, P.bmu) * P.q;
  return min(r, r - P.two_q);
}

__device__ __forceinline__ u32 mulmod(u32 a, u32 b, const DevPrime& P) {
  const u64 x = static_cast<u64>(a) * b;
  const u32 xs = static_cast<u32>(x >> P.bsh);
  u32 r = static_cast<u32>(x) - __umulhi(xs, P.bmu) * P.q;
  r = min(r, r - P.two_q);  // [0, 3q) -> [0, 2q)
  return csub(r, P.q);
}

// Butterfly sum.  HG_BFLY_ALU_ADD: issued as one VIADDMNMX (ALU pipe) so that ptxas cannot
// turn it into IMAD.IADD on the fma pipe, which bounds the transforms.
__device__ __forceinline__ u32 bfly_add(u32 a, u32 b) {
#if HG_BFLY_ALU_ADD
  u32 r;
  asm("{\n\t.reg .u32 t;\n\tadd.u32 t, %1, %2;\n\tmin.u32 %0, t, %3;\n\t}" : "=r"(r) : "r"(a), "r"(b), "r"(0xFFFFFFFFu));
  return r;
#else
  return a + b;
#endif
}

__device__ __forceinline__ u32 addmod(u32 a, u32 b, u32 q) { return csub(a + b, q); }
__device__ __forceinline__ u32 submod(u32 a, u32 b, u32 q) { return csub(a + q - b, q); }

// u32 -> double with the 2^52 pair trick (MOV + DADD), not the slow I2F.F64 (conversion pipe).
__device__ __forceinline__ double u32_to_f64(u32 x) {
  return __dsub_rn(__hiloint2double(0x43300000, static_cast<int>(x)), 4503599627370496.0);
}

// Signed value |c| < q -> residue in [0, q).
__device__ __forceinline__ u32 from_signed(i32 c, u32 q) {
  return c < 0 ? static_cast<u32>(c + static_cast<i32>(q)) : static_cast<u32>(c);
}

// Centered rounding remainder used by divide_round_last (henet/ckks.hpp:132-154):
// r = (x + floor(p/2)) mod p, returned as r - floor(p/2)  (in (-p/2, p/2]).
__device__ __forceinline__ i32 centered_round_rem(u32 x, const DevPrime& P) {
  const u32 r = csub(x + P.half, P.q);
  return static_cast<i32>(r) - static_cast<i32>(P.half);
}

// ---------------------------------------------------------------------------
// Tensor memory as per-thread scratch.  A CTA of T threads takes 64 * T / 128 TMEM
// columns; warp w owns lanes 32 (w % 4) .. + 32 and columns 64 (w / 4) .. + 64, so every
// thread has 64 private 32-bit cells (its lane) that tcgen05.ld / st move 8 at a time.
// Keeping a kernel's per-thread rows there instead of in shared memory frees the shared
// memory that otherwise limits it to 2 CTAs per SM.
// ---------------------------------------------------------------------------
__device__ __forceinline__ u32 tm_smem_addr(const void* p) { return static_cast<u32>(__cvta_generic_to_shared(p)); }

// CELLS (64 or 32) private cells per thread: a kernel that needs fewer takes fewer columns,
// which leaves room for CTAs of other kernels (other streams) on the same SM.
template <int T, int CELLS = 64>
struct TmemScratch {
  static_assert(CELLS == 64 || CELLS == 32, "cells per thread");
  // warps w and w + 4 share TMEM lanes, so a CTA needs CELLS columns per group of 4 warps
  // (rounded up: a CTA of 32 or 64 threads still needs CELLS columns)
  static constexpr u32 kCols = CELLS * ((T + 127) / 128) < 32 ? 32 : CELLS * ((T + 127) / 128);
  u32 base;  // this thread's cell 0: lane | column
  // warp 0 allocates; every thread learns the base after the barrier (slot: one smem word)
  __device__ __forceinline__ void alloc(u32* slot, u32 tid) {
    if (tid < 32) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(tm_smem_addr(slot)),
                   "r"(kCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
    const u32 w = tid >> 5;
#if HG_DEBUG_CHECKS
    if (((*slot) >> 16) != 0 || ((*slot) & 0xFFFFu) + kCols > 512u) __trap();  // self-check build
#endif
    base = *slot + (((w & 3) * 32) << 16) + (w >> 2) * CELLS;
  }
  __device__ __forceinline__ void free(u32 tid) {
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(base & 0xFFFFu), "r"(kCols));
  }
  __device__ __forceinline__ void ld8(u32 col, u32 (&r)[8]) const {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(base + col));
  }
  __device__ __forceinline__ void st8(u32 col, const u32 (&r)[8]) const {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(base + col),
                 "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
  }
  __device__ __forceinline__ static void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
  __device__ __forceinline__ static void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
};

// ---------------------------------------------------------------------------
// NTT block: one CTA of T = N/32 threads transforms one limb held as 32
// registers per thread, in three register passes separated by two shared
// memory exchanges.  Register layouts (tid in [0, T), k in [0, 32)):
//   A : j = tid | k << LOGT                     (natural order, coalesced)
//   B : j = (tid & CBm) | (k & MBm) << CB | (tid >> CB) << LOGT | (k >> MB) << (LOGT + MB)
//   C : j = (k & CBm) | tid << CB | (k >> CB) << (CB + LOGT)
// Forward:  A --(stages LOGN-1..LOGT)--> smem --> B --(LOGT-1..CB)--> smem --> C --(CB-1..0)
// Inverse runs the same passes backwards: C -> B -> A.
// ---------------------------------------------------------------------------
#ifndef HG_NTT_SPLIT
#define HG_NTT_SPLIT 1
#endif
// Pass-B twiddle holder: a row of 32 (w, shoup) pairs in 16 x 128-bit registers, or a
// pointer to the row staged in shared memory (TWS).
template <bool TWS>
struct NttTwB;
template <>
struct NttTwB<false> {
  uint4 r[16];
  __device__ __forceinline__ uint2 at(int n) const {
    return (n & 1) ? make_uint2(r[n >> 1].z, r[n >> 1].w) : make_uint2(r[n >> 1].x, r[n >> 1].y);
  }
};
template <>
struct NttTwB<true> {
  const uint4* row4;  // 16-byte-aligned row in shared memory
  mutable uint4 cur;  // the pair holding slots (2i, 2i+1); stages start at even slots
  __device__ __forceinline__ uint2 at(int slot) const {
    if ((slot & 1) == 0) cur = row4[slot >> 1];
    return (slot & 1) ? make_uint2(cur.z, cur.w) : make_uint2(cur.x, cur.y);
  }
};

// TWS: pass-B twiddles staged in shared memory (64 fewer registers per thread, 31 LDS.64
// per transform): the choice of kernels that gain a CTA per SM from it.
template <int LOGN_, bool TWS = false>
struct Ntt {
  static constexpr int LOGN = LOGN_;
  static constexpr int N = 1 << LOGN;
  static constexpr int LOGT = LOGN - 5;
  static constexpr int T = 1 << LOGT;
  static constexpr int CB = (LOGN >= 14) ? (LOGN - 10) : 3;
  static constexpr int MB = LOGT - CB;
  static constexpr u32 CBm = (1u << CB) - 1;
  static constexpr u32 MBm = (1u << MB) - 1;
  static_assert(LOGN >= 10 && LOGN <= 15, "supported ring degrees: 2^10 .. 2^15");
  static_assert(MB >= 1 && MB <= 5 && CB <= 5, "bad pass split");

  __device__ static __forceinline__ u32 jA(u32 tid, u32 k) { return tid | (k << LOGT); }
  __device__ static __forceinline__ u32 jB(u32 tid, u32 k) {
    return (tid & CBm) | ((k & MBm) << CB) | ((tid >> CB) << LOGT) | ((k >> MB) << (LOGT + MB));
  }
  __device__ static __forceinline__ u32 jC(u32 tid, u32 k) {
    return (k & CBm) | (tid << CB) | ((k >> CB) << (CB + LOGT));
  }
  template <int L>
  __device__ static __forceinline__ u32 jmap(u32 tid, u32 k) {
    if constexpr (L == 0) return jA(tid, k);
    else if constexpr (L == 1) return jB(tid, k);
    else return jC(tid, k);
  }

  // Shared-memory word of element j: one pad word per 32.  Bank-conflict free
  // for all three layouts at N = 2^13, 2^14 (tests/test_ntt_layout.py), and
  // since jmap(tid, k) = base(tid) | const(k) with disjoint bits, the address
  // splits into base(tid) + const(k): every access is an immediate offset.
  static constexpr int XCHG_WORDS = N + (N >> 5);  // exchange buffer
  __device__ static __forceinline__ u32 swz(u32 j) { return j + (j >> 5); }
  // Pass-B twiddles staged (TWS) after the exchange buffer, T >> CB rows padded to 34
  // pairs: 16-byte aligned for 128-bit pair loads, and the 4 rows a warp touches start
  // 4 banks apart.
  static constexpr int TWB_ROWS = T >> CB;
  static constexpr int TWB_STRIDE = 34;
  static constexpr int TWB_WORDS = TWS ? TWB_ROWS * TWB_STRIDE * 2 : 0;
  static constexpr int SMEM_WORDS = XCHG_WORDS + TWB_WORDS;

  // jmap<L>(tid, k) == tpart<L>(tid) | kpart<L>(k) with disjoint bit fields.
  template <int L>
  __device__ static __forceinline__ u32 tpart(u32 tid) {
    if constexpr (L == 0) return tid;
    else if constexpr (L == 1) return (tid & CBm) | ((tid >> CB) << LOGT);
    else return tid << CB;
  }
  template <int L>
  __device__ static __forceinline__ constexpr u32 kpart(u32 k) {
    if constexpr (L == 0) return k << LOGT;
    else if constexpr (L == 1) return ((k & MBm) << CB) | ((k >> MB) << (LOGT + MB));
    else return (k & CBm) | ((k >> CB) << (CB + LOGT));
  }

  template <int L>
  __device__ static __forceinline__ void store(const u32 (&x)[32], u32* sm, u32 tid) {
    u32* base = sm + swz(tpart<L>(tid));
#pragma unroll
    for (int k = 0; k < 32; ++k) base[swz(kpart<L>(k))] = x[k];
  }
  template <int L>
  __device__ static __forceinline__ void load(u32 (&x)[32], const u32* sm, u32 tid) {
    const u32* base = sm + swz(tpart<L>(tid));
#pragma unroll
    for (int k = 0; k < 32; ++k) x[k] = base[swz(kpart<L>(k))];
  }

  // Butterfly bits of pass L occupy register bits [0, NB); the j bit of
  // register bit 0 is BLO.
  template <int L>
  struct PassShape {
    static constexpr int NB = (L == 0) ? 5 : (L == 1 ? MB : CB);
    static constexpr int BLO = (L == 0) ? LOGT : (L == 1 ? CB : 0);
  };

  using TwB = NttTwB<TWS>;
  // Row of staged pass-B twiddles for this thread's group (rows of 32 pairs in global).
  // The shared-memory variant is ordered before pass B by the transform's first barrier,
  // and the previous transform finished reading it before its last barrier.
  // stage = false reuses the rows staged earlier for the same prime and direction (the key
  // switch stages once with stage_rowsB and runs all its forward transforms under one prime).
  __device__ static __forceinline__ void stage_rowsB(const uint2* base, u32* sm, u32 tid) {
    static_assert(TWS, "staging needs the shared-memory twiddle variant");
    uint2* st = reinterpret_cast<uint2*>(sm + XCHG_WORDS);
#pragma unroll
    for (int i = 0; i < TWB_ROWS * 32 / T; ++i) {
      const u32 e = tid + i * T;
      st[(e >> 5) * TWB_STRIDE + (e & 31)] = __ldg(base + e);
    }
  }
  __device__ static __forceinline__ void load_rowB(TwB& tw, const uint2* base, u32* sm, u32 tid, bool stage = true) {
    if constexpr (TWS) {
      uint2* st = reinterpret_cast<uint2*>(sm + XCHG_WORDS);
      if (stage) {
#pragma unroll
        for (int i = 0; i < TWB_ROWS * 32 / T; ++i) {
          const u32 e = tid + i * T;
          st[(e >> 5) * TWB_STRIDE + (e & 31)] = __ldg(base + e);
        }
      }
      tw.row4 = reinterpret_cast<const uint4*>(st + (tid >> CB) * TWB_STRIDE);
    } else {
      (void)sm;
      const uint4* row = reinterpret_cast<const uint4*>(base + static_cast<size_t>(tid >> CB) * 32);
#pragma unroll
      for (int i = 0; i < 16; ++i) tw.r[i] = __ldg(row + i);
    }
  }
  // Pass C's twiddles factor as V(b, c, g) * T_b(tid).  Rather than one extra product by
  // T_b per butterfly (3 x 16 per transform), the registers carry the T factors as a
  // scale: register k of a forward pass C starts multiplied by F_k = prod_{b in bits(k)}
  // T_b, so at stage b every Y holds exactly one more T_b than its X partner and the
  // butterfly needs only V; the stage leaves both outputs at X's scale, and after the last
  // stage every scale is 1.  The inverse (Gentleman-Sande) pass C drops T_b from its
  // products the same way and multiplies register k by F_k at the end.  2^CB - 1 products
  // per group of 2^CB registers instead of CB * 2^(CB-1): 28 instead of 48 at N = 2^13.
  static constexpr int FC = 1 << CB;
  __device__ static __forceinline__ void load_F(uint2 (&f)[FC], const uint2* F, u32 tid) {
    const uint2* row = F + static_cast<size_t>(tid) * FC;
#pragma unroll
    for (int kk = 1; kk < FC; ++kk) f[kk] = __ldg(row + kk);
  }
  __device__ static __forceinline__ void apply_F(u32 (&x)[32], const uint2 (&f)[FC], u32 q) {
#pragma unroll
    for (int kk = 1; kk < FC; ++kk)
#pragma unroll
      for (int g = 0; g < 32 / FC; ++g) x[g * FC + kk] = mul_shoup_lazy(x[g * FC + kk], f[kk].x, f[kk].y, q);
  }
  __device__ static __forceinline__ void scale_C(u32 (&x)[32], const uint2* F, u32 tid, u32 q) {
    uint2 f[FC];
    load_F(f, F, tid);
    apply_F(x, f, q);
  }

  // Forward (Cooley-Tukey, Harvey lazy) stages of pass L.  Values in [0, 4q).
  // Pass A twiddles come from the parameter block, pass B from the preloaded
  // row, pass C as V * T_b(tid) (two Shoup multiplications, no loads).
  template <int L>
  __device__ static __forceinline__ void fwd_pass(u32 (&x)[32], const DevPrime& P, const TwB& twB) {
    constexpr int NB = PassShape<L>::NB;
    constexpr int BLO = PassShape<L>::BLO;
    const u32 q = P.q, q2 = P.two_q;
    int n = 0;
    int slot = 0;  // pass-B row slot: every stage starts at an even slot (128-bit pair loads)
#pragma unroll
    for (int s = 0; s < NB; ++s) {
      const int rb = NB - 1 - s;  // register bit of this stage
      const int b = BLO + rb;     // j bit of this stage (t = 2^b)
      slot = (slot + 1) & ~1;
#if HG_NTT_SPLIT
      // all 16 products of the stage first (independent IMAD.HI chains), then the adds
      u32 Tm[16];
      int m = 0;
#pragma unroll
      for (int g = 0; g < (1 << (5 - NB)); ++g) {
#pragma unroll
        for (int hi = 0; hi < (1 << (NB - 1 - rb)); ++hi) {
          const u32 kh = (static_cast<u32>(g) << NB) | (static_cast<u32>(hi) << (rb + 1));
          const uint2 w = (L == 0) ? P.twA[(1u << (LOGN - 1 - b)) + (kh >> (rb + 1))]
                                   : (L == 1 ? twB.at(slot) : P.tvC[n]);
          ++n;
          ++slot;
#pragma unroll
          for (int lo = 0; lo < (1 << rb); ++lo) {
            const u32 Y = x[(kh | lo) | (1 << rb)];
            Tm[m++] = mul_shoup_lazy(Y, w.x, w.y, q);
          }
        }
      }
      m = 0;
#pragma unroll
      for (int g = 0; g < (1 << (5 - NB)); ++g) {
#pragma unroll
        for (int hi = 0; hi < (1 << (NB - 1 - rb)); ++hi) {
          const u32 kh = (static_cast<u32>(g) << NB) | (static_cast<u32>(hi) << (rb + 1));
#pragma unroll
          for (int lo = 0; lo < (1 << rb); ++lo) {
            const int k0 = kh | lo;
            const int k1 = k0 | (1 << rb);
            u32 X = x[k0];
            X = min(X, X - q2);
            x[k0] = bfly_add(X, Tm[m]);
            x[k1] = X - Tm[m] + q2;
            ++m;
          }
        }
      }
#else
#pragma unroll
      for (int g = 0; g < (1 << (5 - NB)); ++g) {
#pragma unroll
        for (int hi = 0; hi < (1 << (NB - 1 - rb)); ++hi) {
          const u32 kh = (static_cast<u32>(g) << NB) | (static_cast<u32>(hi) << (rb + 1));
          const uint2 w = (L == 0) ? P.twA[(1u << (LOGN - 1 - b)) + (kh >> (rb + 1))]
                                   : (L == 1 ? twB.at(slot) : P.tvC[n]);
          ++n;
          ++slot;
#pragma unroll
          for (int lo = 0; lo < (1 << rb); ++lo) {
            const int k0 = kh | lo;
            const int k1 = k0 | (1 << rb);
            u32 X = x[k0];
            X = min(X, X - q2);
            const u32 Y = x[k1];
            const u32 Tm = mul_shoup_lazy(Y, w.x, w.y, q);
            x[k0] = X + Tm;
            x[k1] = X - Tm + q2;
          }
        }
      }
#endif
    }
  }

  // Inverse (Gentleman-Sande, Harvey lazy) stages of pass L.  Values in [0, 2q).
  // Pass A carries the final stage (m = 1), which also applies N^-1.
  template <int L>
  __device__ static __forceinline__ void inv_pass(u32 (&x)[32], const DevPrime& P, const TwB& twB) {
    constexpr int NB = PassShape<L>::NB;
    constexpr int BLO = PassShape<L>::BLO;
    const u32 q = P.q, q2 = P.two_q;
    int n = 0;
    int slot = 0;
#pragma unroll
    for (int s = 0; s < NB; ++s) {
      const int rb = s;
      const int b = BLO + rb;
      slot = (slot + 1) & ~1;
#pragma unroll
      for (int g = 0; g < (1 << (5 - NB)); ++g) {
#pragma unroll
        for (int hi = 0; hi < (1 << (NB - 1 - rb)); ++hi) {
          const u32 kh = (static_cast<u32>(g) << NB) | (static_cast<u32>(hi) << (rb + 1));
          if (b == LOGN - 1) {
#pragma unroll
            for (int lo = 0; lo < (1 << rb); ++lo) {
              const int k0 = kh | lo;
              const int k1 = k0 | (1 << rb);
              const u32 U = x[k0], V = x[k1];
              x[k0] = mul_shoup_lazy(U + V, P.ninv, P.ninv_sh, q);
              x[k1] = mul_shoup_lazy(U - V + q2, P.w1n, P.w1n_sh, q);
            }
          } else {
            const uint2 w = (L == 0) ? P.itwA[(1u << (LOGN - 1 - b)) + (kh >> (rb + 1))]
                                     : (L == 1 ? twB.at(slot) : P.itvC[n]);
            ++n;
            ++slot;
#pragma unroll
            for (int lo = 0; lo < (1 << rb); ++lo) {
              const int k0 = kh | lo;
              const int k1 = k0 | (1 << rb);
              const u32 U = x[k0], V = x[k1];
              u32 S = U + V;
              x[k0] = min(S, S - q2);
              const u32 D = U - V + q2;
              x[k1] = mul_shoup_lazy(D, w.x, w.y, q);
            }
          }
        }
      }
    }
  }

  // Full forward transform.  In: layout A, values < 4q.  Out: layout C,
  // canonical.  `sm` must hold SMEM_WORDS u32; the call begins and ends with a
  // barrier-protected exchange so the buffer may be reused immediately.
  __device__ static __forceinline__ void forward(u32 (&x)[32], u32* sm, u32 tid, const DevPrime& P,
                                                 bool stage_twiddles = true) {
    TwB twB;
    load_rowB(twB, P.fwdB, sm, tid, stage_twiddles);  // in flight during pass A
    fwd_pass<0>(x, P, twB);
    HG_NTT_SYNC();
#if !HG_T_NOXCHG
    store<0>(x, sm, tid);
#endif
    HG_NTT_SYNC();
#if !HG_T_NOXCHG
    load<1>(x, sm, tid);
#endif
    fwd_pass<1>(x, P, twB);
#if !HG_T_NOXCHG
    store<1>(x, sm, tid);
#endif
    uint2 f[FC];
#if !HG_T_NOF
    load_F(f, P.fwdT, tid);  // while x is in shared memory: the loads cross the barrier
#endif
    HG_NTT_SYNC();
#if !HG_T_NOXCHG
    load<2>(x, sm, tid);
#endif
#if !HG_T_NOF
    apply_F(x, f, P.q);
#endif
    fwd_pass<2>(x, P, twB);
    const u32 q = P.q, q2 = P.two_q;
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      u32 v = x[k];
      v = min(v, v - q2);
      x[k] = min(v, v - q);
    }
  }

  // Full inverse transform.  In: layout C, values < 2q.  Out: layout A, canonical.
  __device__ static __forceinline__ void inverse(u32 (&x)[32], u32* sm, u32 tid, const DevPrime& P) {
    TwB twB;
    load_rowB(twB, P.invB, sm, tid);  // in flight during pass C
    inv_pass<2>(x, P, twB);
    scale_C(x, P.invT, tid, P.q);
    __syncthreads();
    store<2>(x, sm, tid);
    __syncthreads();
    load<1>(x, sm, tid);
    inv_pass<1>(x, P, twB);
    store<1>(x, sm, tid);
    __syncthreads();
    load<0>(x, sm, tid);
    inv_pass<0>(x, P, twB);
    const u32 q = P.q;
#pragma unroll
    for (int k = 0; k < 32; ++k) x[k] = csub(x[k], q);
  }

  // Global memory helpers for one limb row.
  __device__ static __forceinline__ void gload_A(u32 (&x)[32], const u32* __restrict__ row, u32 tid) {
#pragma unroll
    for (int k = 0; k < 32; ++k) x[k] = __ldg(&row[jA(tid, k)]);
  }
  __device__ static __forceinline__ void gstore_A(const u32 (&x)[32], u32* __restrict__ row, u32 tid) {
#pragma unroll
    for (int k = 0; k < 32; ++k) row[jA(tid, k)] = x[k];
  }
  // Thread-major scratch layout "P" (for buffers only these kernels read back): thread
  // tid's registers 4c..4c+3 form the 128-bit word c * T + tid, so each access is a
  // fully coalesced LDG/STG.128.  Register k holds the same coefficient as in layout A.
  template <typename W>
  __device__ static __forceinline__ void gload_P(W (&x)[32], const W* __restrict__ row, u32 tid) {
    static_assert(sizeof(W) == 4, "32-bit words");
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(row) + c * T + tid);
      x[4 * c] = static_cast<W>(v.x); x[4 * c + 1] = static_cast<W>(v.y);
      x[4 * c + 2] = static_cast<W>(v.z); x[4 * c + 3] = static_cast<W>(v.w);
    }
  }
  template <typename W>
  __device__ static __forceinline__ void gstore_P(const W (&x)[32], W* __restrict__ row, u32 tid) {
    static_assert(sizeof(W) == 4, "32-bit words");
#pragma unroll
    for (int c = 0; c < 8; ++c)
      reinterpret_cast<uint4*>(row)[c * T + tid] =
          make_uint4(static_cast<u32>(x[4 * c]), static_cast<u32>(x[4 * c + 1]), static_cast<u32>(x[4 * c + 2]),
                     static_cast<u32>(x[4 * c + 3]));
  }
  // Layout C groups of 2^CB consecutive words -> 128-bit accesses.
  __device__ static __forceinline__ void gload_C(u32 (&x)[32], const u32* __restrict__ row, u32 tid) {
#pragma unroll
    for (int k = 0; k < 32; k += 4) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(row + jC(tid, k)));
      x[k] = v.x; x[k + 1] = v.y; x[k + 2] = v.z; x[k + 3] = v.w;
    }
  }
  __device__ static __forceinline__ void gstore_C(const u32 (&x)[32], u32* __restrict__ row, u32 tid) {
#pragma unroll
    for (int k = 0; k < 32; k += 4) {
      *reinterpret_cast<uint4*>(row + jC(tid, k)) = make_uint4(x[k], x[k + 1], x[k + 2], x[k + 3]);
    }
  }
};

}  // namespace hg
