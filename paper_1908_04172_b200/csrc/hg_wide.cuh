// SPDX-License-Identifier: Apache-2.0
//
// "Wide" residue arithmetic: contexts whose basis contains a prime >= 2^30
// (BASELINE configs 4 / 5b: N = 2^14, chain [40, 30 x 7] bits + 40-bit special)
// store every residue as u64.  Same algorithms and index conventions as the u32
// path (hg_device.cuh); arithmetic follows the reference's 128-bit Barrett
// reduction (henet/modmath.hpp:122-140) and 64-bit Shoup butterflies (values in
// [0, 4q) < 2^64 for q < 2^62).
#pragma once

#include "hg_device.cuh"

namespace hg {

struct DevPrimeW {
  u64 q, two_q, half;
  u64 r128_lo, r128_hi;  // floor(2^128 / q) as (low, high) words, henet/modmath.hpp:91-115
  u64 ninv, ninv_sh;     // N^-1 and floor(ninv * 2^64 / q)
  u64 w1n, w1n_sh;       // inv_root_powers[1] * N^-1
  u64 t64;               // 2^64 mod q
  const ulonglong2* fwd; // N entries (psi^bitrev(i), shoup64), natural index
  const ulonglong2* inv;
};

struct BasisW {
  DevPrimeW p[kMaxPrimes];
  // Host pointer to the context's u32 Basis (Ntt<> tables for every prime < 2^32): launchers
  // run the limbs below 2^30 on the u32 transforms with u64 I/O.  Not read on the device.
  const void* narrow;
};

__device__ __forceinline__ u64 csub64(u64 x, u64 q) { return x >= q ? x - q : x; }

// barrett_reduce_128 of the reference, verbatim semantics (canonical result).
__device__ __forceinline__ u64 barrett128(u64 z_lo, u64 z_hi, const DevPrimeW& P) {
  const u64 r0 = P.r128_lo, r1 = P.r128_hi;
  u64 carry = __umul64hi(z_lo, r0);
  u64 prod_lo = z_lo * r1, prod_hi = __umul64hi(z_lo, r1);
  u64 tmp1 = prod_lo + carry;
  u64 tmp3 = prod_hi + (tmp1 < prod_lo ? 1 : 0);
  prod_lo = z_hi * r0;
  prod_hi = __umul64hi(z_hi, r0);
  const u64 s = tmp1 + prod_lo;
  carry = prod_hi + (s < tmp1 ? 1 : 0);
  tmp1 = z_hi * r1 + tmp3 + carry;
  const u64 r = z_lo - tmp1 * P.q;
  return r >= P.q ? r - P.q : r;
}

// Any u64 -> [0, q) for q < 2^62: Barrett with the 64-bit mu = floor(2^64 / q) (r128_hi);
// the estimate is at most 2 below floor(x / q), so two conditional subtractions finish it.
__device__ __forceinline__ u64 red64(u64 x, const DevPrimeW& P) {
  const u64 r = x - __umul64hi(x, P.r128_hi) * P.q;
  const u64 r1 = r >= P.q ? r - P.q : r;
  return r1 >= P.q ? r1 - P.q : r1;
}

// Primes below 2^31 (the 30-bit limbs of a wide context): operands < 2q keep the product
// below 2^64, so one 64-bit Barrett replaces the 128-bit one.  The branch is uniform per limb.
__device__ __forceinline__ u64 mulmod_w(u64 a, u64 b, const DevPrimeW& P) {
  if (P.q < (1ull << 31)) return red64(a * b, P);
  return barrett128(a * b, __umul64hi(a, b), P);
}

__device__ __forceinline__ u64 addmod_w(u64 a, u64 b, u64 q) { return csub64(a + b, q); }

__device__ __forceinline__ u64 mul_shoup64_lazy(u64 x, u64 w, u64 wsh, u64 q) {
  return x * w - __umul64hi(x, wsh) * q;  // [0, 2q)
}
__device__ __forceinline__ u64 mul_shoup64(u64 x, u64 w, u64 wsh, u64 q) {
  return csub64(mul_shoup64_lazy(x, w, wsh, q), q);
}

using i64 = int64_t;

__device__ __forceinline__ i64 centered_round_rem_w(u64 x, const DevPrimeW& P) {
  const u64 r = csub64(x + P.half, P.q);
  return static_cast<i64>(r) - static_cast<i64>(P.half);
}

// residue of a signed value (|c| < 2^63), any relation to q
__device__ __forceinline__ u64 signed_residue_w(i64 c, const DevPrimeW& P) {
  const u64 m = barrett128(static_cast<u64>(c < 0 ? -c : c), 0, P);
  return (c < 0 && m != 0) ? P.q - m : m;
}

// u64 NTT block: same three register passes / layouts as Ntt<LOGN>, twiddles from
// the natural-order table (psi^bitrev(m + i)).
template <int LOGN_>
struct NttW {
  using NT = Ntt<LOGN_>;
  static constexpr int LOGN = LOGN_, N = NT::N, LOGT = NT::LOGT, T = NT::T, CB = NT::CB, MB = NT::MB;
  static constexpr int SMEM_WORDS = NT::XCHG_WORDS;  // u64 words

  template <int L>
  __device__ static __forceinline__ void store(const u64 (&x)[32], u64* sm, u32 tid) {
    u64* base = sm + NT::swz(NT::template tpart<L>(tid));
#pragma unroll
    for (int k = 0; k < 32; ++k) base[NT::swz(NT::template kpart<L>(k))] = x[k];
  }
  template <int L>
  __device__ static __forceinline__ void load(u64 (&x)[32], const u64* sm, u32 tid) {
    const u64* base = sm + NT::swz(NT::template tpart<L>(tid));
#pragma unroll
    for (int k = 0; k < 32; ++k) x[k] = base[NT::swz(NT::template kpart<L>(k))];
  }

  template <int L>
  __device__ static __forceinline__ void fwd_pass(u64 (&x)[32], u32 tid, const DevPrimeW& P) {
    constexpr int NB = NT::template PassShape<L>::NB;
    constexpr int BLO = NT::template PassShape<L>::BLO;
    const u64 q = P.q, q2 = P.two_q;
#pragma unroll
    for (int s = 0; s < NB; ++s) {
      const int rb = NB - 1 - s;
      const int b = BLO + rb;
#pragma unroll
      for (int g = 0; g < (1 << (5 - NB)); ++g) {
#pragma unroll
        for (int hi = 0; hi < (1 << (NB - 1 - rb)); ++hi) {
          const u32 kh = (static_cast<u32>(g) << NB) | (static_cast<u32>(hi) << (rb + 1));
          const u32 j = NT::template jmap<L>(tid, kh);
          const ulonglong2 w = __ldg(&P.fwd[(1u << (LOGN - 1 - b)) + (j >> (b + 1))]);
#pragma unroll
          for (int lo = 0; lo < (1 << rb); ++lo) {
            const int k0 = kh | lo, k1 = k0 | (1 << rb);
            u64 X = x[k0];
            X = X >= q2 ? X - q2 : X;
            const u64 Tm = mul_shoup64_lazy(x[k1], w.x, w.y, q);
            x[k0] = X + Tm;
            x[k1] = X - Tm + q2;
          }
        }
      }
    }
  }

  template <int L>
  __device__ static __forceinline__ void inv_pass(u64 (&x)[32], u32 tid, const DevPrimeW& P) {
    constexpr int NB = NT::template PassShape<L>::NB;
    constexpr int BLO = NT::template PassShape<L>::BLO;
    const u64 q = P.q, q2 = P.two_q;
#pragma unroll
    for (int s = 0; s < NB; ++s) {
      const int rb = s;
      const int b = BLO + rb;
#pragma unroll
      for (int g = 0; g < (1 << (5 - NB)); ++g) {
#pragma unroll
        for (int hi = 0; hi < (1 << (NB - 1 - rb)); ++hi) {
          const u32 kh = (static_cast<u32>(g) << NB) | (static_cast<u32>(hi) << (rb + 1));
          if (b == LOGN - 1) {
#pragma unroll
            for (int lo = 0; lo < (1 << rb); ++lo) {
              const int k0 = kh | lo, k1 = k0 | (1 << rb);
              const u64 U = x[k0], V = x[k1];
              x[k0] = mul_shoup64_lazy(U + V, P.ninv, P.ninv_sh, q);
              x[k1] = mul_shoup64_lazy(U - V + q2, P.w1n, P.w1n_sh, q);
            }
          } else {
            const u32 j = NT::template jmap<L>(tid, kh);
            const ulonglong2 w = __ldg(&P.inv[(1u << (LOGN - 1 - b)) + (j >> (b + 1))]);
#pragma unroll
            for (int lo = 0; lo < (1 << rb); ++lo) {
              const int k0 = kh | lo, k1 = k0 | (1 << rb);
              const u64 U = x[k0], V = x[k1];
              const u64 S = U + V;
              x[k0] = S >= q2 ? S - q2 : S;
              x[k1] = mul_shoup64_lazy(U - V + q2, w.x, w.y, q);
            }
          }
        }
      }
    }
  }

  __device__ static __forceinline__ void forward(u64 (&x)[32], u64* sm, u32 tid, const DevPrimeW& P) {
    fwd_pass<0>(x, tid, P);
    __syncthreads();
    store<0>(x, sm, tid);
    __syncthreads();
    load<1>(x, sm, tid);
    fwd_pass<1>(x, tid, P);
    store<1>(x, sm, tid);
    __syncthreads();
    load<2>(x, sm, tid);
    fwd_pass<2>(x, tid, P);
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      u64 v = x[k];
      v = v >= P.two_q ? v - P.two_q : v;
      x[k] = csub64(v, P.q);
    }
  }

  __device__ static __forceinline__ void inverse(u64 (&x)[32], u64* sm, u32 tid, const DevPrimeW& P) {
    inv_pass<2>(x, tid, P);
    __syncthreads();
    store<2>(x, sm, tid);
    __syncthreads();
    load<1>(x, sm, tid);
    inv_pass<1>(x, tid, P);
    store<1>(x, sm, tid);
    __syncthreads();
    load<0>(x, sm, tid);
    inv_pass<0>(x, tid, P);
#pragma unroll
    for (int k = 0; k < 32; ++k) x[k] = csub64(x[k], P.q);
  }

  __device__ static __forceinline__ void gload_A(u64 (&x)[32], const u64* __restrict__ row, u32 tid) {
#pragma unroll
    for (int k = 0; k < 32; ++k) x[k] = __ldg(&row[NT::jA(tid, k)]);
  }
  __device__ static __forceinline__ void gstore_A(const u64 (&x)[32], u64* __restrict__ row, u32 tid) {
#pragma unroll
    for (int k = 0; k < 32; ++k) row[NT::jA(tid, k)] = x[k];
  }
  __device__ static __forceinline__ void gload_C(u64 (&x)[32], const u64* __restrict__ row, u32 tid) {
#pragma unroll
    for (int k = 0; k < 32; k += 2) {
      const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(row + NT::jC(tid, k)));
      x[k] = v.x;
      x[k + 1] = v.y;
    }
  }
  __device__ static __forceinline__ void gstore_C(const u64 (&x)[32], u64* __restrict__ row, u32 tid) {
#pragma unroll
    for (int k = 0; k < 32; k += 2)
      *reinterpret_cast<ulonglong2*>(row + NT::jC(tid, k)) = make_ulonglong2(x[k], x[k + 1]);
  }
};

}  // namespace hg
