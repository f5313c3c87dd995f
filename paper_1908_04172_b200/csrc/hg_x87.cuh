// SPDX-License-Identifier: Apache-2.0
//
// Exact emulation of the reference's encoding rounding on the GPU:
//   roundl((long double)value * (long double)scale)   (henet/encoding.hpp:122-126, 184)
// x87 extended precision = 64-bit mantissa, round-to-nearest-even; the exact
// 106-bit product of the two double mantissas is rounded to 64 bits the same
// way, then rounded half away from zero to an integer magnitude.
#pragma once

#include <cstdint>

#include "hg_device.cuh"

namespace hg {

struct X87 {
  bool neg;
  unsigned long long mant;  // 64-bit normalized mantissa (0 for zero)
  int exp;                  // value = mant * 2^exp
};

__device__ __forceinline__ void split_double(double v, unsigned long long& m, int& e) {
  const unsigned long long bits = __double_as_longlong(v) & 0x7fffffffffffffffull;
  const int be = static_cast<int>(bits >> 52);
  const unsigned long long frac = bits & ((1ull << 52) - 1);
  if (be == 0) { m = frac; e = -1074; }
  else { m = frac | (1ull << 52); e = be - 1075; }
}

__device__ __forceinline__ X87 x87_mul(double a, double b) {
  X87 r;
  r.neg = (__double_as_longlong(a) ^ __double_as_longlong(b)) < 0;
  unsigned long long ma, mb;
  int ea, eb;
  split_double(a, ma, ea);
  split_double(b, mb, eb);
  if (ma == 0 || mb == 0) { r.mant = 0; r.exp = 0; r.neg = false; return r; }
  unsigned __int128 p = static_cast<unsigned __int128>(ma) * mb;
  int e = ea + eb;
  const unsigned long long hi = static_cast<unsigned long long>(p >> 64);
  const int nb = hi ? 128 - __clzll(hi) : 64 - __clzll(static_cast<unsigned long long>(p));
  if (nb > 64) {
    const int sh = nb - 64;
    unsigned __int128 m = p >> sh;
    const unsigned __int128 rem = p & ((static_cast<unsigned __int128>(1) << sh) - 1);
    const unsigned __int128 halfv = static_cast<unsigned __int128>(1) << (sh - 1);
    if (rem > halfv || (rem == halfv && (m & 1))) m += 1;
    e += sh;
    if (m >> 64) { m >>= 1; e += 1; }
    r.mant = static_cast<unsigned long long>(m);
  } else {
    const int sh = 64 - nb;  // normalize
    r.mant = static_cast<unsigned long long>(p) << sh;
    e -= sh;
  }
  r.exp = e;
  return r;
}

// roundl (half away from zero) of |x| as a 128-bit magnitude.
__device__ __forceinline__ unsigned __int128 x87_roundl_mag(const X87& x) {
  if (x.mant == 0) return 0;
  if (x.exp >= 0) return static_cast<unsigned __int128>(x.mant) << x.exp;
  const int s = -x.exp;
  if (s > 65) return 0;
  const unsigned __int128 m = x.mant;
  return (m + (static_cast<unsigned __int128>(1) << (s - 1))) >> s;
}

__device__ __forceinline__ u32 residue_mag(unsigned __int128 mag, bool neg, const DevPrime& P) {
  // Barrett (reduce64) instead of u64 '%': (hi mod q) 2^64 + lo, with 2^64 mod q =
  // (2^32 mod q)^2 mod q; every partial product stays below 2^64 for q < 2^32
  const u64 hi = static_cast<u64>(mag >> 64), lo = static_cast<u64>(mag);
  u32 r = reduce64(lo, P);
  if (hi != 0) {
    const u32 t64 = reduce64(static_cast<u64>(P.r32) * P.r32, P);
    r = reduce64(static_cast<u64>(reduce64(hi, P)) * t64 + r, P);
  }
  if (neg && r != 0) r = P.q - r;
  return r;
}

// |roundl(v * s)| as a 128-bit magnitude plus its sign.
__device__ __forceinline__ unsigned __int128 x87_round_product(double v, double s, bool& neg) {
  const X87 x = x87_mul(v, s);
  neg = x.neg;
  return x87_roundl_mag(x);
}

}  // namespace hg
