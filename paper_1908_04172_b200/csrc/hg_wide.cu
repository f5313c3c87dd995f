// SPDX-License-Identifier: Apache-2.0
//
// u64 ("wide") kernels for contexts with primes >= 2^30 (BASELINE configs 4/5b).
// Same algorithms as the u32 kernels of hg_kernels.cu; every result canonical.
#include <cuda_runtime.h>

#include "hg_wide.hpp"

namespace hg {

// ---------------------------------------------------------------------------
// Batched NTT / INTT
// ---------------------------------------------------------------------------
// Limbs [lo, lo + cnt) of every row of `level` limbs; one CTA per (row, limb).
template <int LOGN, bool INV>
__global__ void __launch_bounds__(1 << (LOGN - 5), 1) k_ntt_w(u64* data, u32 level, u32 lo, u32 cnt, BasisW B) {
  using NT = NttW<LOGN>;
  extern __shared__ u64 smw[];
  const u32 tid = threadIdx.x;
  const u64 ct = blockIdx.x / cnt;
  const u32 limb = lo + blockIdx.x % cnt;
  const DevPrimeW& P = B.p[limb];
  u64* r = data + (ct * level + limb) * NT::N;
  u64 x[32];
  if (!INV) {
    NT::gload_A(x, r, tid);
    NT::forward(x, smw, tid, P);
    NT::gstore_C(x, r, tid);
  } else {
    NT::gload_C(x, r, tid);
    NT::inverse(x, smw, tid, P);
    NT::gstore_A(x, r, tid);
  }
}

// The limbs below 2^30 of a wide tensor on the u32 transform (Ntt<>, one Shoup product per
// butterfly on 32-bit words instead of the 64-bit Shoup of NttW): residues are narrowed on
// load and widened on store, in place.  Limbs [lo, level) of every row.
template <int LOGN, bool INV>
__global__ void __launch_bounds__(1 << (LOGN - 5), (LOGN <= 13 ? 4 : HG_NTT14_MINB)) k_ntt_w32(u64* data, u32 level, u32 lo, Basis B) {
  using NT = Ntt<LOGN, true>;
  extern __shared__ u32 sm32[];
  const u32 tid = threadIdx.x;
  const u32 cnt = level - lo;
  const u64 ct = blockIdx.x / cnt;
  const u32 limb = lo + blockIdx.x % cnt;
  const DevPrime& P = B.p[limb];
  u64* r = data + (ct * level + limb) * NT::N;
  u32 x[32];
  if (!INV) {
#pragma unroll
    for (int k = 0; k < 32; ++k) x[k] = static_cast<u32>(__ldg(&r[NT::jA(tid, k)]));
    NT::forward(x, sm32, tid, P);
#pragma unroll
    for (int k = 0; k < 32; k += 4) {
      ulonglong2* o = reinterpret_cast<ulonglong2*>(r + NT::jC(tid, k));
      o[0] = make_ulonglong2(x[k], x[k + 1]);
      o[1] = make_ulonglong2(x[k + 2], x[k + 3]);
    }
  } else {
#pragma unroll
    for (int k = 0; k < 32; k += 4) {
      const ulonglong2* in = reinterpret_cast<const ulonglong2*>(r + NT::jC(tid, k));
      const ulonglong2 a = __ldg(in), b = __ldg(in + 1);
      x[k] = static_cast<u32>(a.x);
      x[k + 1] = static_cast<u32>(a.y);
      x[k + 2] = static_cast<u32>(b.x);
      x[k + 3] = static_cast<u32>(b.y);
    }
    NT::inverse(x, sm32, tid, P);
#pragma unroll
    for (int k = 0; k < 32; ++k) r[NT::jA(tid, k)] = x[k];
  }
}

// encrypt's c0 = NTT(e) - a s + pt (henet/ckks.hpp:235-239) fused into the error's forward NTT
// for the limbs below 2^30: the transformed error never goes back to HBM.
template <int LOGN>
__global__ void __launch_bounds__(1 << (LOGN - 5), (LOGN <= 13 ? 4 : HG_NTT14_MINB))
    k_enc_ntt_w32(u64* ct, const u64* err, const u64* pt, const u64* sk, u32 level, u32 lo, Basis B) {
  using NT = Ntt<LOGN, true>;
  extern __shared__ u32 sm32[];
  const u32 tid = threadIdx.x;
  const u32 cnt = level - lo;
  const u64 e = blockIdx.x / cnt;
  const u32 limb = lo + blockIdx.x % cnt;
  const DevPrime& P = B.p[limb];
  const u64 per = static_cast<u64>(level) * NT::N, row = static_cast<u64>(limb) * NT::N;
  const u64* er = err + e * per + row;
  u32 x[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) x[k] = static_cast<u32>(__ldg(&er[NT::jA(tid, k)]));
  NT::forward(x, sm32, tid, P);
  u64* c0 = ct + e * 2 * per + row;
  const u64* c1 = c0 + per;
  const u64* pr = pt + e * per + row;
  const u64* sr = sk + row;
  auto ld4 = [](const u64* p) {
    const ulonglong2 a = __ldg(reinterpret_cast<const ulonglong2*>(p)), b = __ldg(reinterpret_cast<const ulonglong2*>(p) + 1);
    return make_uint4(static_cast<u32>(a.x), static_cast<u32>(a.y), static_cast<u32>(b.x), static_cast<u32>(b.y));
  };
#pragma unroll
  for (int k = 0; k < 32; k += 4) {
    const u32 j = NT::jC(tid, k);
    const uint4 av = ld4(c1 + j), sv = ld4(sr + j), pv = ld4(pr + j);
    const u32 A[4] = {av.x, av.y, av.z, av.w}, S[4] = {sv.x, sv.y, sv.z, sv.w}, Pt[4] = {pv.x, pv.y, pv.z, pv.w};
    u32 o[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) o[i] = addmod(submod(x[k + i], mulmod(A[i], S[i], P), P.q), Pt[i], P.q);
    ulonglong2* d = reinterpret_cast<ulonglong2*>(c0 + j);
    d[0] = make_ulonglong2(o[0], o[1]);
    d[1] = make_ulonglong2(o[2], o[3]);
  }
}

// decrypt's m = c0 + c1 s (+ c2 s^2) (henet/ckks.hpp:256-268) fused into the INTT of the limbs
// below 2^30: the NTT-domain words are combined in registers (u32 arithmetic) as they are
// loaded, transformed, and only the coefficient-domain m is written -- no m round trip
// through HBM between a combine kernel and the transform.
template <int LOGN>
__global__ void __launch_bounds__(1 << (LOGN - 5), (LOGN <= 13 ? 4 : HG_NTT14_MINB))
    k_dec_intt_w32(const u64* ct, const u64* sk, u64* m, u32 polys, u32 level, u32 lo, Basis B) {
  using NT = Ntt<LOGN, true>;
  extern __shared__ u32 sm32[];
  const u32 tid = threadIdx.x;
  const u32 cnt = level - lo;
  const u64 e = blockIdx.x / cnt;
  const u32 limb = lo + blockIdx.x % cnt;
  const DevPrime& P = B.p[limb];
  const u64 per = static_cast<u64>(level) * NT::N;
  const u64* c0 = ct + e * polys * per + static_cast<u64>(limb) * NT::N;
  const u64* sr = sk + static_cast<u64>(limb) * NT::N;
  u32 x[32];
  auto ld4 = [](const u64* p) {
    const ulonglong2 a = __ldg(reinterpret_cast<const ulonglong2*>(p)), b = __ldg(reinterpret_cast<const ulonglong2*>(p) + 1);
    return make_uint4(static_cast<u32>(a.x), static_cast<u32>(a.y), static_cast<u32>(b.x), static_cast<u32>(b.y));
  };
#pragma unroll
  for (int k = 0; k < 32; k += 4) {
    const u32 j = NT::jC(tid, k);
    const uint4 a0 = ld4(c0 + j), a1 = ld4(c0 + per + j), sv = ld4(sr + j);
    const u32 A0[4] = {a0.x, a0.y, a0.z, a0.w}, A1[4] = {a1.x, a1.y, a1.z, a1.w}, S[4] = {sv.x, sv.y, sv.z, sv.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) x[k + i] = addmod(A0[i], mulmod(A1[i], S[i], P), P.q);
    if (polys == 3) {
      const uint4 a2 = ld4(c0 + 2 * per + j);
      const u32 A2[4] = {a2.x, a2.y, a2.z, a2.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) x[k + i] = addmod(x[k + i], mulmod(A2[i], mulmod(S[i], S[i], P), P), P.q);
    }
  }
  NT::inverse(x, sm32, tid, P);
  u64* out = m + (e * level + limb) * NT::N;
#pragma unroll
  for (int k = 0; k < 32; ++k) out[NT::jA(tid, k)] = x[k];
}

// ---------------------------------------------------------------------------
// Rescale (henet/ckks.hpp:504-519), NTT-domain form as in k_rescale.
// ---------------------------------------------------------------------------
template <int LOGN>
__global__ void __launch_bounds__(1 << (LOGN - 5), 1) k_rescale_w(RescaleArgsW a, BasisW B) {
  using NT = NttW<LOGN>;
  constexpr int N = NT::N;
  constexpr int T = NT::T;
  extern __shared__ u64 smw[];
  i32* cs = reinterpret_cast<i32*>(smw + NT::SMEM_WORDS);  // |correction| < p_last/2 < 2^31 (p < 2^32)
  i64* cg = a.corr64 ? a.corr64 + blockIdx.x * static_cast<u64>(N) : nullptr;  // p >= 2^32: global row
  const u32 tid = threadIdx.x;
  const u64 row = blockIdx.x;
  const u32 L = a.level;
  const u64* src = a.in + row * L * N;
  u64* dst = a.out + row * (L - 1) * N;
  u64 x[32];
  {
    const DevPrimeW& Pl = B.p[L - 1];
    NT::gload_C(x, src + static_cast<u64>(L - 1) * N, tid);
    NT::inverse(x, smw, tid, Pl);
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      const i64 c = centered_round_rem_w(x[k], Pl);
      if (cg) cg[k * T + tid] = c;
      else cs[k * T + tid] = static_cast<i32>(c);
    }
  }
  const u32 kept = a.limb_cnt ? a.limb_cnt : L - 1;
  for (u32 i = 0; i < kept; ++i) {
    const DevPrimeW& Pi = B.p[i];
#pragma unroll
    for (int k = 0; k < 32; ++k) x[k] = signed_residue_w(cg ? cg[k * T + tid] : cs[k * T + tid], Pi);
    NT::forward(x, smw, tid, Pi);
    const u64 q = Pi.q, pv = a.pinv[i], ps = a.pinv_sh[i];
    const u64* in_i = src + static_cast<u64>(i) * N;
    u64* out_i = dst + static_cast<u64>(i) * N;
#pragma unroll
    for (int k = 0; k < 32; k += 2) {
      const u32 j = NT::NT::jC(tid, k);
      const ulonglong2 y = __ldg(reinterpret_cast<const ulonglong2*>(in_i + j));
      *reinterpret_cast<ulonglong2*>(out_i + j) =
          make_ulonglong2(mul_shoup64(y.x + q - x[k], pv, ps, q), mul_shoup64(y.y + q - x[k + 1], pv, ps, q));
    }
  }
}

// ---------------------------------------------------------------------------
// Dense / conv modular contraction with 128-bit accumulation for wide limbs
// (products up to 2^80) and the u64 lazy path (with folding) for narrow limbs.
// ---------------------------------------------------------------------------
struct Acc128 {
  u64 lo, hi;
};
__device__ __forceinline__ void mac128(Acc128& a, u64 x, u64 w) {
  asm("mad.lo.cc.u64 %0, %2, %3, %0;\n\tmadc.hi.u64 %1, %2, %3, %1;" : "+l"(a.lo), "+l"(a.hi) : "l"(x), "l"(w));
}

constexpr int kWBK = 16, kWTM = 4, kWBN = 128, kWWarps = 8;

__global__ void __launch_bounds__(kWWarps * 32) k_mac_dense_w(MacDenseArgsW a, BasisW B) {
  __shared__ __align__(16) u64 xs[kWBK][kWBN];
  __shared__ __align__(16) u64 ws[kWBK][kWTM * kWWarps];
  const u32 tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const u32 BM = kWTM * kWWarps;
  const u32 n0 = blockIdx.x * kWBN;
  const u32 m0 = blockIdx.y * BM;
  const u32 nl = a.limb_cnt ? a.limb_cnt : a.level;
  const u32 poly = blockIdx.z / nl, limb = a.limb_lo + blockIdx.z % nl;
  const DevPrimeW& P = B.p[limb];
  const bool wide = P.q >= (1ull << 32);
  const u64 xstride = static_cast<u64>(a.polys) * a.x_level * a.N;
  const u64* Xb = a.X + (static_cast<u64>(poly) * a.x_level + limb) * a.N + n0;
  const u64* Wb = a.W + static_cast<u64>(limb) * a.K * a.Mpad + m0;
  Acc128 acc[kWTM][4];
#pragma unroll
  for (int i = 0; i < kWTM; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = {0, 0};
  for (u32 k0 = 0; k0 < a.K; k0 += kWBK) {
    for (u32 c = tid; c < kWBK * kWBN; c += blockDim.x) {
      const u32 r = c / kWBN, col = c % kWBN, k = k0 + r;
      xs[r][col] = k < a.K ? __ldg(Xb + static_cast<u64>(k) * xstride + col) : 0;
    }
    for (u32 c = tid; c < kWBK * BM; c += blockDim.x) {
      const u32 r = c / BM, col = c % BM, k = k0 + r;
      ws[r][col] = k < a.K ? __ldg(Wb + static_cast<u64>(k) * a.Mpad + col) : 0;
    }
    __syncthreads();
    if (wide) {
#pragma unroll 4
      for (int kk = 0; kk < kWBK; ++kk) {
        const ulonglong2 x01 = *reinterpret_cast<const ulonglong2*>(&xs[kk][lane * 4]);
        const ulonglong2 x23 = *reinterpret_cast<const ulonglong2*>(&xs[kk][lane * 4 + 2]);
#pragma unroll
        for (int i = 0; i < kWTM; ++i) {
          const u64 w = ws[kk][warp * kWTM + i];
          mac128(acc[i][0], x01.x, w);
          mac128(acc[i][1], x01.y, w);
          mac128(acc[i][2], x23.x, w);
          mac128(acc[i][3], x23.y, w);
        }
      }
      if (a.fold[limb]) {
        // primes near 2^62: r + 16 (q-1)^2 < 2^128 only after a reduction per k-tile
#pragma unroll
        for (int i = 0; i < kWTM; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = {barrett128(acc[i][j].lo, acc[i][j].hi, P), 0};
      }
    } else {
      // narrow limb stored wide: 32x32 products into the low word, folded every 8 taps
      const u64 r32 = static_cast<u64>((1ull << 32) % P.q);
#pragma unroll 4
      for (int kk = 0; kk < kWBK; ++kk) {
        const ulonglong2 x01 = *reinterpret_cast<const ulonglong2*>(&xs[kk][lane * 4]);
        const ulonglong2 x23 = *reinterpret_cast<const ulonglong2*>(&xs[kk][lane * 4 + 2]);
#pragma unroll
        for (int i = 0; i < kWTM; ++i) {
          const u32 w = static_cast<u32>(ws[kk][warp * kWTM + i]);
          acc[i][0].lo += static_cast<u64>(w) * static_cast<u32>(x01.x);
          acc[i][1].lo += static_cast<u64>(w) * static_cast<u32>(x01.y);
          acc[i][2].lo += static_cast<u64>(w) * static_cast<u32>(x23.x);
          acc[i][3].lo += static_cast<u64>(w) * static_cast<u32>(x23.y);
        }
        if ((kk & 7) == 7) {
#pragma unroll
          for (int i = 0; i < kWTM; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j].lo = (acc[i][j].lo & 0xffffffffull) + (acc[i][j].lo >> 32) * r32;
        }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < kWTM; ++i) {
    const u32 m = m0 + warp * kWTM + i;
    if (m >= a.M) continue;
    const u64 bv = (a.bias != nullptr && poly == 0) ? __ldg(&a.bias[static_cast<u64>(limb) * a.Mpad + m]) : 0;
    u64* yp = a.Y + ((static_cast<u64>(m) * a.polys + poly) * a.level + limb) * a.N + n0 + lane * 4;
    u64 o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) o[j] = addmod_w(barrett128(acc[i][j].lo, acc[i][j].hi, P), bv, P.q);
    *reinterpret_cast<ulonglong2*>(yp) = make_ulonglong2(o[0], o[1]);
    *reinterpret_cast<ulonglong2*>(yp + 2) = make_ulonglong2(o[2], o[3]);
  }
}

constexpr int kWMaxTaps = 1024;
constexpr int kWFT = 8;

// Window taps in ascending (c, ky, kx) order with the padding skipped (henet/graph.hpp:976-989),
// walked by every thread (uniform control flow, no serial tap-list prologue).
template <typename F>
__device__ __forceinline__ void for_each_tap(const MacConvArgsW& a, u32 oy, u32 ox, F&& body) {
  for (u32 c = 0; c < a.C; ++c)
    for (u32 ky = 0; ky < a.win; ++ky) {
      const int iy = static_cast<int>(oy * a.stride + ky) - static_cast<int>(a.pad_top);
      if (iy < 0 || iy >= static_cast<int>(a.IH)) continue;
      for (u32 kx = 0; kx < a.win; ++kx) {
        const int ix = static_cast<int>(ox * a.stride + kx) - static_cast<int>(a.pad_left);
        if (ix < 0 || ix >= static_cast<int>(a.IW)) continue;
        body((c * a.IH + static_cast<u32>(iy)) * a.IW + static_cast<u32>(ix), (c * a.win + ky) * a.win + kx);
      }
    }
}

__global__ void __launch_bounds__(128) k_mac_conv_w(MacConvArgsW a, BasisW B) {
  const u32 tid = threadIdx.x;
  const u32 pos = blockIdx.y;
  const u32 oy = pos / a.OW, ox = pos % a.OW;
  const u32 nchunks = (a.F + kWFT - 1) / kWFT;
  const u32 per_group = a.polys * a.level * nchunks;
  const u32 g = blockIdx.z / per_group, zz = blockIdx.z % per_group;
  a.X += g * a.gx;
  a.Y += g * a.gy;
  a.W += g * a.gw;
  if (a.bias != nullptr) a.bias += g * a.gb;
  const u32 pl = zz / nchunks;
  const u32 f0 = (zz % nchunks) * kWFT;
  const u32 poly = pl / a.level, limb = pl % a.level;
  const DevPrimeW& P = B.p[limb];
  const u32 n = (blockIdx.x * blockDim.x + tid) * 2;
  const u32 taps_all = a.C * a.win * a.win;
  const u64 xstride = static_cast<u64>(a.polys) * a.x_level * a.N;
  const u64* Xb = a.X + (static_cast<u64>(poly) * a.x_level + limb) * a.N + n;
  const u64* Wl = a.W + static_cast<u64>(limb) * a.F * taps_all;
  auto store = [&](int f, u64 v0, u64 v1) {
    const u32 ff = f0 + f;
    const u64 bv = (a.bias != nullptr && poly == 0) ? __ldg(&a.bias[static_cast<u64>(limb) * a.F + ff]) : 0;
    const u64 e = static_cast<u64>(ff) * a.OH * a.OW + pos;
    u64* yp = a.Y + ((e * a.polys + poly) * a.level + limb) * a.N + n;
    *reinterpret_cast<ulonglong2*>(yp) = make_ulonglong2(addmod_w(v0, bv, P.q), addmod_w(v1, bv, P.q));
  };
  if (P.q < (1ull << 30)) {
    // a limb below 2^30 (the 30-bit limbs of c4/c5b): one 32 x 32 -> 64 IMAD.WIDE per MAC
    // (products < 2^60), folded (acc = lo + hi * (2^32 mod q) < 2^62 + 2^32) every 8 taps, so
    // the sums stay below 2^64
    const u64 r32 = (1ull << 32) % P.q;
    u64 acc[kWFT][2];
#pragma unroll
    for (int f = 0; f < kWFT; ++f) acc[f][0] = acc[f][1] = 0;
    u32 cnt = 0;
    for_each_tap(a, oy, ox, [&](u32 tin, u32 tw) {
      const ulonglong2 xv = __ldg(reinterpret_cast<const ulonglong2*>(Xb + static_cast<u64>(tin) * xstride));
      const u32 x0 = static_cast<u32>(xv.x), x1 = static_cast<u32>(xv.y);
#pragma unroll
      for (int f = 0; f < kWFT; ++f) {
        if (f0 + f >= a.F) break;
        const u32 w = static_cast<u32>(__ldg(&Wl[static_cast<u64>(f0 + f) * taps_all + tw]));
        acc[f][0] += static_cast<u64>(x0) * w;
        acc[f][1] += static_cast<u64>(x1) * w;
      }
      if ((++cnt & 7) == 0) {
#pragma unroll
        for (int f = 0; f < kWFT; ++f)
#pragma unroll
          for (int j = 0; j < 2; ++j) acc[f][j] = (acc[f][j] & 0xffffffffull) + (acc[f][j] >> 32) * r32;
      }
    });
#pragma unroll
    for (int f = 0; f < kWFT; ++f)
      if (f0 + f < a.F) store(f, barrett128(acc[f][0], 0, P), barrett128(acc[f][1], 0, P));
    return;
  }
  Acc128 acc[kWFT][2];
#pragma unroll
  for (int f = 0; f < kWFT; ++f) acc[f][0] = acc[f][1] = {0, 0};
  const bool fold = a.fold[limb] != 0;
  u32 cnt = 0;
  for_each_tap(a, oy, ox, [&](u32 tin, u32 tw) {
    const ulonglong2 xv = __ldg(reinterpret_cast<const ulonglong2*>(Xb + static_cast<u64>(tin) * xstride));
#pragma unroll
    for (int f = 0; f < kWFT; ++f) {
      if (f0 + f >= a.F) break;
      const u64 w = __ldg(&Wl[static_cast<u64>(f0 + f) * taps_all + tw]);
      mac128(acc[f][0], xv.x, w);
      mac128(acc[f][1], xv.y, w);
    }
    if (fold && (++cnt & 7) == 0) {  // primes near 2^62: keep r + 8 (q-1)^2 < 2^128
#pragma unroll
      for (int f = 0; f < kWFT; ++f)
#pragma unroll
        for (int j = 0; j < 2; ++j) acc[f][j] = {barrett128(acc[f][j].lo, acc[f][j].hi, P), 0};
    }
  });
#pragma unroll
  for (int f = 0; f < kWFT; ++f)
    if (f0 + f < a.F)
      store(f, barrett128(acc[f][0].lo, acc[f][0].hi, P), barrett128(acc[f][1].lo, acc[f][1].hi, P));
}

// Grouped 1 -> 1 convolutions (a depthwise layer, MacConvArgsW::groups = C, C = F = 1 per
// group): one thread per (group, poly, limb, coefficient pair) walks every output position,
// so its window weights are loaded once and the overlapping windows of neighbouring outputs
// are re-read from L1 -- instead of one 128-thread CTA per (position, slice) with nine loads
// each (the tap-gather k_mac_conv_w).  Same sums: taps in (ky, kx) order, padding skipped,
// 30-bit limbs as u64 IMAD.WIDE sums folded every 8 taps, wider limbs in 128 bits.
// WIN: the window (3 for MobileNetV2), compile-time.  Along each output row the thread keeps
// the WIN x WIN input window in registers and slides it one column per output (WIN new loads
// instead of WIN^2); taps outside the input enter as zeros, which add nothing to the exact
// sums (the tap-gather kernel skips them), so the results are the same residues.
template <int WIN>
__global__ void __launch_bounds__(128) k_dwconv_w(MacConvArgsW a, BasisW B) {
  constexpr int T2 = WIN * WIN;
  const u32 g = blockIdx.z;
  const u32 poly = blockIdx.y / a.level, limb = blockIdx.y % a.level;
  const u32 n = (blockIdx.x * blockDim.x + threadIdx.x) * 2;
  if (n >= a.N) return;
  const DevPrimeW& P = B.p[limb];
  const u64* X = a.X + g * a.gx + (static_cast<u64>(poly) * a.x_level + limb) * a.N + n;
  const u64 xstride = static_cast<u64>(a.polys) * a.x_level * a.N;  // words per input element
  u64* Y = a.Y + g * a.gy + (static_cast<u64>(poly) * a.level + limb) * a.N + n;
  const u64 ystride = static_cast<u64>(a.polys) * a.level * a.N;
  u64 w[T2];
#pragma unroll
  for (int t = 0; t < T2; ++t) w[t] = __ldg(&a.W[g * a.gw + limb * T2 + t]);
  const u64 bv = (a.bias != nullptr && poly == 0) ? __ldg(&a.bias[g * a.gb + limb]) : 0;
  const bool narrow = P.q < (1ull << 30);
  const u64 r32 = narrow ? (1ull << 32) % P.q : 0;
  const bool fold = a.fold[limb] != 0;
  auto ld = [&](int iy, int ix) {
    if (iy < 0 || iy >= static_cast<int>(a.IH) || ix < 0 || ix >= static_cast<int>(a.IW))
      return make_ulonglong2(0, 0);
    return __ldg(reinterpret_cast<const ulonglong2*>(X + (static_cast<u64>(iy) * a.IW + static_cast<u32>(ix)) * xstride));
  };
  for (u32 oy = 0; oy < a.OH; ++oy) {
    const int iy0 = static_cast<int>(oy * a.stride) - static_cast<int>(a.pad_top);
    const int ix00 = -static_cast<int>(a.pad_left);
    ulonglong2 xw[WIN][WIN];  // [ky][kx] window of the current output
#pragma unroll
    for (int ky = 0; ky < WIN; ++ky)
#pragma unroll
      for (int kx = 0; kx < WIN; ++kx) xw[ky][kx] = ld(iy0 + ky, ix00 + kx);
    for (u32 ox = 0; ox < a.OW; ++ox) {
      if (ox > 0) {  // slide: stride columns shift in (stride 1 for MobileNetV2)
        const int ixn = static_cast<int>(ox * a.stride) - static_cast<int>(a.pad_left);
        if (a.stride == 1) {
#pragma unroll
          for (int ky = 0; ky < WIN; ++ky) {
#pragma unroll
            for (int kx = 0; kx + 1 < WIN; ++kx) xw[ky][kx] = xw[ky][kx + 1];
            xw[ky][WIN - 1] = ld(iy0 + ky, ixn + WIN - 1);
          }
        } else {
#pragma unroll
          for (int ky = 0; ky < WIN; ++ky)
#pragma unroll
            for (int kx = 0; kx < WIN; ++kx) xw[ky][kx] = ld(iy0 + ky, ixn + kx);
        }
      }
      u64 s0 = 0, s1 = 0;
      Acc128 c0{0, 0}, c1{0, 0};
      u32 cnt = 0;
#pragma unroll
      for (int ky = 0; ky < WIN; ++ky)
#pragma unroll
        for (int kx = 0; kx < WIN; ++kx) {
          const ulonglong2 xv = xw[ky][kx];
          const u64 wt = w[ky * WIN + kx];
          if (narrow) {
            s0 += static_cast<u64>(static_cast<u32>(xv.x)) * static_cast<u32>(wt);
            s1 += static_cast<u64>(static_cast<u32>(xv.y)) * static_cast<u32>(wt);
            if (T2 > 8 && (++cnt & 7) == 0) {
              s0 = (s0 & 0xffffffffull) + (s0 >> 32) * r32;
              s1 = (s1 & 0xffffffffull) + (s1 >> 32) * r32;
            }
          } else {
            mac128(c0, xv.x, wt);
            mac128(c1, xv.y, wt);
            if (T2 > 8 && fold && (++cnt & 7) == 0) {
              c0 = {barrett128(c0.lo, c0.hi, P), 0};
              c1 = {barrett128(c1.lo, c1.hi, P), 0};
            }
          }
        }
      u64 o0, o1;
      if (narrow) {
        o0 = red64(s0, P);
        o1 = red64(s1, P);
      } else {
        o0 = barrett128(c0.lo, c0.hi, P);
        o1 = barrett128(c1.lo, c1.hi, P);
      }
      *reinterpret_cast<ulonglong2*>(Y + static_cast<u64>(oy * a.OW + ox) * ystride) =
          make_ulonglong2(addmod_w(o0, bv, P.q), addmod_w(o1, bv, P.q));
    }
  }
}

// Depthwise with the whole (channel, poly, limb) input tile of 64 coefficients staged in
// shared memory (IH IW x 64 u64, 51 KB for the c4 10 x 10 tile): every input word is read
// from HBM once (the per-thread walk of k_dwconv_w re-read rows from DRAM once the CTAs in
// flight outgrew L2), then warp w computes outputs w, w + 8, ... from shared memory, lane =
// coefficient pair (512 contiguous bytes per warp load and store).  Same exact sums.
// MODE (block-uniform, chosen per limb): 0 = primes < 2^30, u64 IMAD.WIDE sums folded every
// 8 taps; 1 = primes <= 2^40 (c4's limb 0) as 20-bit halves, x w = xl wl + (xl wh + xh wl)
// 2^20 + xh wh 2^40 with every partial sum of <= 25 products < 2^46 in a u64 (four
// IMAD.WIDE.U32 per tap); 2 = any prime, 128-bit sums.
template <int WIN, int MODE>
__device__ __forceinline__ void dw_outputs(const MacConvArgsW& a, const DevPrimeW& P, const ulonglong2* dws,
                                           const u64 (&w)[WIN * WIN], u64 bv, u64* Y, u64 ystride, u32 lane,
                                           u32 grp) {
  constexpr int T2 = WIN * WIN;
  const u64 r32 = MODE == 0 ? (1ull << 32) % P.q : 0;
  const u32 nout = a.OH * a.OW;
  u32 oy = grp / a.OW, ox = grp % a.OW;  // advanced incrementally (no division per output)
  for (u32 o = grp; o < nout; o += 8) {
    const int iy0 = static_cast<int>(oy * a.stride) - static_cast<int>(a.pad_top);
    const int ix0 = static_cast<int>(ox * a.stride) - static_cast<int>(a.pad_left);
    bool rok[WIN], cok[WIN];
#pragma unroll
    for (int k = 0; k < WIN; ++k) {
      rok[k] = static_cast<u32>(iy0 + k) < a.IH;
      cok[k] = static_cast<u32>(ix0 + k) < a.IW;
    }
    const int base = iy0 * static_cast<int>(a.IW) + ix0;
    u64 s0 = 0, s1 = 0, m0 = 0, m1 = 0, h0 = 0, h1 = 0;
    Acc128 c0{0, 0}, c1{0, 0};
    u32 cnt = 0;
#pragma unroll
    for (int ky = 0; ky < WIN; ++ky) {
      const int rowb = base + ky * static_cast<int>(a.IW);
#pragma unroll
      for (int kx = 0; kx < WIN; ++kx) {
        const bool ok = rok[ky] && cok[kx];  // a padding tap adds zero
        const ulonglong2 xv = ok ? dws[static_cast<u32>(rowb + kx) * 32 + lane] : make_ulonglong2(0, 0);
        const u64 wt = w[ky * WIN + kx];
        if constexpr (MODE == 0) {
          s0 += static_cast<u64>(static_cast<u32>(xv.x)) * static_cast<u32>(wt);
          s1 += static_cast<u64>(static_cast<u32>(xv.y)) * static_cast<u32>(wt);
          if (T2 > 8 && (++cnt & 7) == 0) {
            s0 = (s0 & 0xffffffffull) + (s0 >> 32) * r32;
            s1 = (s1 & 0xffffffffull) + (s1 >> 32) * r32;
          }
        } else if constexpr (MODE == 1) {
          const u32 wl = static_cast<u32>(wt & 0xFFFFF), wh = static_cast<u32>(wt >> 20);
          const u32 al = static_cast<u32>(xv.x & 0xFFFFF), ah = static_cast<u32>(xv.x >> 20);
          const u32 bl = static_cast<u32>(xv.y & 0xFFFFF), bh = static_cast<u32>(xv.y >> 20);
          s0 += static_cast<u64>(al) * wl;
          m0 += static_cast<u64>(al) * wh + static_cast<u64>(ah) * wl;
          h0 += static_cast<u64>(ah) * wh;
          s1 += static_cast<u64>(bl) * wl;
          m1 += static_cast<u64>(bl) * wh + static_cast<u64>(bh) * wl;
          h1 += static_cast<u64>(bh) * wh;
        } else {
          mac128(c0, xv.x, wt);
          mac128(c1, xv.y, wt);
          if (T2 > 8 && (++cnt & 7) == 0) {  // keep r + 8 (q-1)^2 < 2^128 for primes near 2^62
            c0 = {barrett128(c0.lo, c0.hi, P), 0};
            c1 = {barrett128(c1.lo, c1.hi, P), 0};
          }
        }
      }
    }
    u64 o0, o1;
    if constexpr (MODE == 0) {
      o0 = red64(s0, P);
      o1 = red64(s1, P);
    } else if constexpr (MODE == 1) {
      // l + m 2^20 + h 2^40 as (lo, hi) words, then the reference's 128-bit Barrett
      auto join = [&](u64 l, u64 m, u64 h) {
        const u64 ml = m << 20, mh = m >> 44, hl = h << 40, hh = h >> 24;
        const u64 lo = l + ml;
        u64 hi = mh + (lo < ml ? 1 : 0);
        const u64 lo2 = lo + hl;
        hi += hh + (lo2 < hl ? 1 : 0);
        return barrett128(lo2, hi, P);
      };
      o0 = join(s0, m0, h0);
      o1 = join(s1, m1, h1);
    } else {
      o0 = barrett128(c0.lo, c0.hi, P);
      o1 = barrett128(c1.lo, c1.hi, P);
    }
    *reinterpret_cast<ulonglong2*>(Y + static_cast<u64>(o) * ystride) =
        make_ulonglong2(addmod_w(o0, bv, P.q), addmod_w(o1, bv, P.q));
    ox += 8;
    while (ox >= a.OW) {
      ox -= a.OW;
      ++oy;
    }
  }
}

template <int WIN>
__global__ void __launch_bounds__(256) k_dwconv_ws(MacConvArgsW a, BasisW B) {
  extern __shared__ ulonglong2 dws[];  // [IH IW][32] coefficient pairs
  constexpr int T2 = WIN * WIN;
  const u32 g = blockIdx.z;
  const u32 poly = blockIdx.y / a.level, limb = blockIdx.y % a.level;
  const u32 n0 = blockIdx.x * 64, lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const DevPrimeW& P = B.p[limb];
  const u64 xstride = static_cast<u64>(a.polys) * a.x_level * a.N;
  const u64 ystride = static_cast<u64>(a.polys) * a.level * a.N;
  const u64* X = a.X + g * a.gx + (static_cast<u64>(poly) * a.x_level + limb) * a.N + n0 + 2 * lane;
  u64* Y = a.Y + g * a.gy + (static_cast<u64>(poly) * a.level + limb) * a.N + n0 + 2 * lane;
  const u32 npos = a.IH * a.IW;
  for (u32 pi = grp; pi < npos; pi += 8)
    dws[pi * 32 + lane] = __ldg(reinterpret_cast<const ulonglong2*>(X + static_cast<u64>(pi) * xstride));
  u64 w[T2];
#pragma unroll
  for (int t = 0; t < T2; ++t) w[t] = __ldg(&a.W[g * a.gw + limb * T2 + t]);
  const u64 bv = (a.bias != nullptr && poly == 0) ? __ldg(&a.bias[g * a.gb + limb]) : 0;
  __syncthreads();
  if (P.q < (1ull << 30))
    dw_outputs<WIN, 0>(a, P, dws, w, bv, Y, ystride, lane, grp);
  else if (P.q <= (1ull << 40) && T2 <= 25)
    dw_outputs<WIN, 1>(a, P, dws, w, bv, Y, ystride, lane, grp);
  else
    dw_outputs<WIN, 2>(a, P, dws, w, bv, Y, ystride, lane, grp);
}

// ---------------------------------------------------------------------------
// Element-wise
// ---------------------------------------------------------------------------
__global__ void k_ew_w(EwArgsW a, BasisW B) {
  const u32 N = a.N;
  const u64 rows = a.count * a.polys_out * a.level;
  const u64 tiles_per_row = N / 2;
  const u64 idx = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= rows * tiles_per_row) return;
  const u64 row = idx / tiles_per_row;
  const u32 n = static_cast<u32>(idx % tiles_per_row) * 2;
  const u32 limb = row % a.level;
  const u32 poly = (row / a.level) % a.polys_out;
  const u64 e = row / (static_cast<u64>(a.level) * a.polys_out);
  const DevPrimeW& P = B.p[limb];
  const u64 q = P.q;
  auto ld = [&](const u64* base, u32 polys, u32 p) {
    return *reinterpret_cast<const ulonglong2*>(base + ((e * polys + p) * a.level + limb) * N + n);
  };
  ulonglong2 o;
  switch (a.op) {
    case EwOp::AddCC: {
      const ulonglong2 x = ld(a.a, a.polys_a, poly), y = ld(a.b, a.polys_a, poly);
      o = make_ulonglong2(addmod_w(x.x, y.x, q), addmod_w(x.y, y.y, q));
      break;
    }
    case EwOp::MulScalar: {
      const ulonglong2 x = ld(a.a, a.polys_a, poly);
      const u64 r = a.res[(a.per_element ? e / a.pt_div : 0) * a.level + limb];
      o = make_ulonglong2(mulmod_w(x.x, r, P), mulmod_w(x.y, r, P));
      break;
    }
    case EwOp::AddScalar: {
      o = ld(a.a, a.polys_a, poly);
      if (poly == 0) {
        const u64 r = a.res[(a.per_element ? e / a.pt_div : 0) * a.level + limb];
        o = make_ulonglong2(addmod_w(o.x, r, q), addmod_w(o.y, r, q));
      }
      break;
    }
    case EwOp::GatherMul: {
      const u32 src = a.gidx[e];
      if (src == 0xFFFFFFFFu) {
        o = make_ulonglong2(0, 0);
      } else {
        const ulonglong2 x =
            *reinterpret_cast<const ulonglong2*>(a.a + ((static_cast<u64>(src) * a.polys_a + poly) * a.level + limb) * N + n);
        const u64 r = a.res[static_cast<u64>(a.gw[e]) * a.level + limb];
        o = make_ulonglong2(mulmod_w(x.x, r, P), mulmod_w(x.y, r, P));
      }
      break;
    }
    case EwOp::AddVector: {
      o = ld(a.a, a.polys_a, poly);
      if (poly == 0) {
        const ulonglong2 y = *reinterpret_cast<const ulonglong2*>(
            a.b + ((a.per_element ? e / a.pt_div : 0) * a.level + limb) * static_cast<u64>(N) + n);
        o = make_ulonglong2(addmod_w(o.x, y.x, q), addmod_w(o.y, y.y, q));
      }
      break;
    }
    case EwOp::Tensor: {
      ulonglong2 x, y;
      if (poly == 0) { x = ld(a.a, 2, 0); y = ld(a.b, 2, 0); }
      else if (poly == 2) { x = ld(a.a, 2, 1); y = ld(a.b, 2, 1); }
      else { x = ld(a.a, 2, 0); y = ld(a.b, 2, 1); }
      o = make_ulonglong2(mulmod_w(x.x, y.x, P), mulmod_w(x.y, y.y, P));
      if (poly == 1) {
        x = ld(a.a, 2, 1);
        y = ld(a.b, 2, 0);
        o.x = addmod_w(o.x, mulmod_w(x.x, y.x, P), q);
        o.y = addmod_w(o.y, mulmod_w(x.y, y.y, P), q);
      }
      break;
    }
    default:
      o = ld(a.a, a.polys_a, poly);
      break;
  }
  *reinterpret_cast<ulonglong2*>(a.out + ((e * a.polys_out + poly) * a.level + limb) * N + n) = o;
}

__global__ void k_validate_w(const u64* w, u64 words, u32 level, u32 N, BasisW B, int* bad) {
  const u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= words) return;
  if (w[i] >= B.p[(i / N) % level].q) atomicExch(bad, 1);
}

// ---------------------------------------------------------------------------
// Scalar encoding with u64 residues (x87 product rounding shared with the u32 path)
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_encode_scalars_w(const T* vals, u64 count, u32 row_len, u32 row_stride, u64 limb_stride,
                                   u32 level, double scale, u64* out, BasisW B) {
  const u64 v = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= count) return;
  bool neg;
  const unsigned __int128 mag = x87_round_product(static_cast<double>(vals[v]), scale, neg);
  const u64 dst = (v / row_len) * row_stride + v % row_len;
  for (u32 i = 0; i < level; ++i) {
    const DevPrimeW& P = B.p[i];
    u64 r = barrett128(static_cast<u64>(mag), static_cast<u64>(mag >> 64), P);
    if (neg && r != 0) r = P.q - r;
    out[i * limb_stride + dst] = r;
  }
}

// ---------------------------------------------------------------------------
// Relinearization (henet/ckks.hpp:442-499) for u64 residues, any primes < 2^62.
// ---------------------------------------------------------------------------
template <int LOGN>
__global__ void __launch_bounds__(1 << (LOGN - 5), 1) k_relin_digits_w(RelinArgsW a, BasisW B) {
  using NT = NttW<LOGN>;
  extern __shared__ u64 smw[];
  const u32 tid = threadIdx.x;
  const u64 ct = blockIdx.x / a.level;
  const u32 j = blockIdx.x % a.level;
  u64 x[32];
  NT::gload_C(x, a.A + ((ct * 3 + 2) * a.level + j) * NT::N, tid);
  NT::inverse(x, smw, tid, B.p[j]);  // c2 limb j to the coefficient domain (:450-451)
  NT::gstore_A(x, a.D + (ct * a.level + j) * NT::N, tid);
}

template <int LOGN>
__global__ void __launch_bounds__(1 << (LOGN - 5), 1) k_relin_keysw_w(RelinArgsW a, BasisW B) {
  using NT = NttW<LOGN>;
  constexpr int N = NT::N;
  extern __shared__ u64 smw[];
  const u32 tid = threadIdx.x;
  const u32 L = a.level;
  const u64 ct = blockIdx.x / (L + 1);
  const u32 t = blockIdx.x % (L + 1);
  const bool special = t == L;
  const u32 bidx = special ? a.chain_len : t;  // the key's special limb sits at chain_len (:448)
  const DevPrimeW& P = B.p[bidx];
  const u64 q = P.q;
  u64* acc0 = a.ACC + ((ct * 2 + 0) * (L + 1) + t) * N;
  u64* acc1 = a.ACC + ((ct * 2 + 1) * (L + 1) + t) * N;
  for (u32 j = 0; j < L; ++j) {
    u64 y[32];
    NT::gload_A(y, a.D + (ct * L + j) * N, tid);
#pragma unroll
    for (int k = 0; k < 32; ++k) y[k] = y[k] < q ? y[k] : barrett128(y[k], 0, P);  // :463
    NT::forward(y, smw, tid, P);
    const u64* k0 = a.key + ((static_cast<u64>(j) * 2 + 0) * (a.chain_len + 1) + bidx) * N;
    const u64* k1 = a.key + ((static_cast<u64>(j) * 2 + 1) * (a.chain_len + 1) + bidx) * N;
#pragma unroll
    for (int k = 0; k < 32; k += 2) {
      const u32 jj = NT::NT::jC(tid, k);  // this thread's own positions: no barrier needed
      const ulonglong2 w0 = __ldg(reinterpret_cast<const ulonglong2*>(k0 + jj));
      const ulonglong2 w1 = __ldg(reinterpret_cast<const ulonglong2*>(k1 + jj));
      ulonglong2 p0 = make_ulonglong2(mulmod_w(y[k], w0.x, P), mulmod_w(y[k + 1], w0.y, P));
      ulonglong2 p1 = make_ulonglong2(mulmod_w(y[k], w1.x, P), mulmod_w(y[k + 1], w1.y, P));
      if (j != 0) {
        const ulonglong2 s0 = *reinterpret_cast<const ulonglong2*>(acc0 + jj);
        const ulonglong2 s1 = *reinterpret_cast<const ulonglong2*>(acc1 + jj);
        p0 = make_ulonglong2(addmod_w(s0.x, p0.x, q), addmod_w(s0.y, p0.y, q));
        p1 = make_ulonglong2(addmod_w(s1.x, p1.x, q), addmod_w(s1.y, p1.y, q));
      }
      *reinterpret_cast<ulonglong2*>(acc0 + jj) = p0;
      *reinterpret_cast<ulonglong2*>(acc1 + jj) = p1;
    }
  }
  if (!special) return;
  // divide_round_last by P (:478-495): r = (INTT(acc_P) + floor(P/2)) mod P, centred
  for (int c = 0; c < 2; ++c) {
    u64 y[32];
    NT::gload_C(y, c ? acc1 : acc0, tid);
    NT::inverse(y, smw, tid, P);
    i64* cr = a.CORR + (ct * 2 + c) * N;
#pragma unroll
    for (int k = 0; k < 32; ++k) cr[NT::NT::jA(tid, k)] = centered_round_rem_w(y[k], P);
  }
}

template <int LOGN>
__global__ void __launch_bounds__(1 << (LOGN - 5), 1) k_relin_moddown_w(RelinArgsW a, BasisW B) {
  using NT = NttW<LOGN>;
  constexpr int N = NT::N;
  extern __shared__ u64 smw[];
  const u32 tid = threadIdx.x;
  const u32 L = a.level;
  const u64 ct = blockIdx.x / (2 * L);
  const u32 poly = (blockIdx.x / L) % 2;
  const u32 i = blockIdx.x % L;
  const DevPrimeW& Pi = B.p[i];
  const u64 q = Pi.q, pv = a.pinvP[i], ps = a.pinvP_sh[i];
  const i64* cr = a.CORR + (ct * 2 + poly) * N;
  u64 z[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) z[k] = signed_residue_w(cr[NT::NT::jA(tid, k)], Pi);
  NT::forward(z, smw, tid, Pi);  // NTT_i(c mod q_i)
  const u64* accp = a.ACC + ((ct * 2 + poly) * (L + 1) + i) * N;
  const u64* dp = a.A + ((ct * 3 + poly) * L + i) * N;
  u64* op = a.out + ((ct * 2 + poly) * L + i) * N;
#pragma unroll
  for (int k = 0; k < 32; k += 2) {
    const u32 jj = NT::NT::jC(tid, k);
    const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(accp + jj));
    const ulonglong2 d = __ldg(reinterpret_cast<const ulonglong2*>(dp + jj));
    // (x_i - c) * P^-1 mod q_i, then + c_poly (add_inplace)
    *reinterpret_cast<ulonglong2*>(op + jj) =
        make_ulonglong2(addmod_w(d.x, mul_shoup64(v.x + q - z[k], pv, ps, q), q),
                        addmod_w(d.y, mul_shoup64(v.y + q - z[k + 1], pv, ps, q), q));
  }
}

// ---------------------------------------------------------------------------
// Launchers
// ---------------------------------------------------------------------------
#define HG_LOGN_SWITCH_W(logn, ...)                  \
  switch (logn) {                                    \
    case 11: { constexpr int LN = 11; __VA_ARGS__; } break; \
    case 12: { constexpr int LN = 12; __VA_ARGS__; } break; \
    case 13: { constexpr int LN = 13; __VA_ARGS__; } break; \
    case 14: { constexpr int LN = 14; __VA_ARGS__; } break; \
    default: return -1;                              \
  }

template <typename K>
static void set_smem_w(K kernel, size_t bytes) {
  if (bytes > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
}

int launch_ntt_w(int logn, u64* data, u64 rows, u32 level, bool inverse, const BasisW& B, cudaStream_t s) {
  if (rows == 0) return 0;
  // limbs [lo, level) below 2^30 go to the u32 transform (HG_NTT_W32=0: all on the u64 one)
  static const bool w32 = [] {
    const char* e = getenv("HG_NTT_W32");
    return !(e != nullptr && e[0] == '0');
  }();
  u32 lo = level;
  if (w32 && B.narrow != nullptr)
    while (lo > 0 && B.p[lo - 1].q < (1ull << 30)) --lo;
  const u64 count = rows / level;
  int launches = 0;
  HG_LOGN_SWITCH_W(logn, {
    if (lo > 0) {
      const size_t sm = sizeof(u64) * NttW<LN>::SMEM_WORDS;
      auto k = inverse ? k_ntt_w<LN, true> : k_ntt_w<LN, false>;
      set_smem_w(k, sm);
      ProfScope ps_("k_ntt_w", s);
      k<<<count * lo, 1 << (LN - 5), sm, s>>>(data, level, 0, lo, B);
      ++launches;
    }
    if (lo < level) {
      const size_t sm = sizeof(u32) * Ntt<LN, true>::SMEM_WORDS;
      auto k = inverse ? k_ntt_w32<LN, true> : k_ntt_w32<LN, false>;
      set_smem_w(k, sm);
      ProfScope ps_("k_ntt_w32", s);
      k<<<count * (level - lo), 1 << (LN - 5), sm, s>>>(data, level, lo, *static_cast<const Basis*>(B.narrow));
      ++launches;
    }
  });
  return launches;
}

u32 wide_narrow_lo(const BasisW& B, u32 level) {
  u32 lo = level;
  if (B.narrow != nullptr)
    while (lo > 0 && B.p[lo - 1].q < (1ull << 30)) --lo;
  return lo;
}

int launch_dec_intt_w(int logn, const u64* ct, const u64* sk, u64* m, u64 count, u32 polys, u32 level,
                      const BasisW& B, cudaStream_t s) {
  const u32 lo = wide_narrow_lo(B, level);
  if (count == 0 || lo >= level || (polys != 2 && polys != 3)) return -2;
  int launches = 0;
  HG_LOGN_SWITCH_W(logn, {
    if (lo > 0) {  // the wide limbs: m already combined (k_dec_combine), INTT on the u64 transform
      const size_t sm = sizeof(u64) * NttW<LN>::SMEM_WORDS;
      set_smem_w(k_ntt_w<LN, true>, sm);
      ProfScope ps_("k_ntt_w", s);
      k_ntt_w<LN, true><<<count * lo, 1 << (LN - 5), sm, s>>>(m, level, 0, lo, B);
      ++launches;
    }
    const size_t sm = sizeof(u32) * Ntt<LN, true>::SMEM_WORDS;
    set_smem_w(k_dec_intt_w32<LN>, sm);
    ProfScope ps_("k_dec_intt_w32", s);
    k_dec_intt_w32<LN><<<count * (level - lo), 1 << (LN - 5), sm, s>>>(ct, sk, m, polys, level, lo,
                                                                       *static_cast<const Basis*>(B.narrow));
    ++launches;
  });
  return launches;
}

int launch_enc_ntt_w(int logn, u64* ct, u64* err, const u64* pt, const u64* sk, u64 count, u32 level,
                     const BasisW& B, cudaStream_t s) {
  const u32 lo = wide_narrow_lo(B, level);
  if (count == 0 || lo >= level) return -2;
  int launches = 0;
  HG_LOGN_SWITCH_W(logn, {
    if (lo > 0) {  // the wide limbs: error NTT'd in place (combined afterwards by k_enc_combine)
      const size_t sm = sizeof(u64) * NttW<LN>::SMEM_WORDS;
      set_smem_w(k_ntt_w<LN, false>, sm);
      ProfScope ps_("k_ntt_w", s);
      k_ntt_w<LN, false><<<count * lo, 1 << (LN - 5), sm, s>>>(err, level, 0, lo, B);
      ++launches;
    }
    const size_t sm = sizeof(u32) * Ntt<LN, true>::SMEM_WORDS;
    set_smem_w(k_enc_ntt_w32<LN>, sm);
    ProfScope ps_("k_enc_ntt_w32", s);
    k_enc_ntt_w32<LN><<<count * (level - lo), 1 << (LN - 5), sm, s>>>(ct, err, pt, sk, level, lo,
                                                                      *static_cast<const Basis*>(B.narrow));
    ++launches;
  });
  return launches;
}

int launch_rescale_w(int logn, const RescaleArgsW& a, const BasisW& B, cudaStream_t s) {
  if (a.rows == 0) return 0;
  HG_LOGN_SWITCH_W(logn, {
    const size_t sm = sizeof(u64) * NttW<LN>::SMEM_WORDS + sizeof(i32) * NttW<LN>::N;
    set_smem_w(k_rescale_w<LN>, sm);
    { ProfScope ps_("k_rescale_w", s);
    k_rescale_w<LN><<<a.rows, 1 << (LN - 5), sm, s>>>(a, B);
    }
  });
  return 1;
}

int launch_relin_w(int logn, const RelinArgsW& a, const BasisW& B, cudaStream_t s) {
  if (a.count == 0) return 0;
  HG_LOGN_SWITCH_W(logn, {
    const size_t sm = sizeof(u64) * NttW<LN>::SMEM_WORDS;
    const u32 T = 1u << (LN - 5);
    set_smem_w(k_relin_digits_w<LN>, sm);
    set_smem_w(k_relin_keysw_w<LN>, sm);
    set_smem_w(k_relin_moddown_w<LN>, sm);
    { ProfScope ps_("k_relin_digits_w", s);
    k_relin_digits_w<LN><<<a.count * a.level, T, sm, s>>>(a, B);
    }
    { ProfScope ps_("k_relin_keysw_w", s);
    k_relin_keysw_w<LN><<<a.count * (a.level + 1), T, sm, s>>>(a, B);
    }
    { ProfScope ps_("k_relin_moddown_w", s);
    k_relin_moddown_w<LN><<<a.count * 2 * a.level, T, sm, s>>>(a, B);
    }
  });
  return 1;
}

u32 mac_dense_w_bm() { return kWTM * kWWarps; }

int launch_mac_dense_w(const MacDenseArgsW& a, const BasisW& B, cudaStream_t s) {
  const u32 BM = kWTM * kWWarps;
  if (a.Mpad % BM != 0 || a.N % kWBN != 0) return -1;
  dim3 grid(a.N / kWBN, (a.M + BM - 1) / BM, a.polys * (a.limb_cnt ? a.limb_cnt : a.level));
  { ProfScope ps_("k_mac_dense_w", s);
  k_mac_dense_w<<<grid, kWWarps * 32, 0, s>>>(a, B);
  }
  return 1;
}

__global__ void k_limbs_to_u32(const u64* __restrict__ in, u32* __restrict__ out, u64 rows, u32 Lw, u32 lo, u32 cnt,
                               u32 N) {
  const u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;  // one u64x2 -> u32x2
  const u64 per_row = static_cast<u64>(cnt) * N / 2;
  if (i >= rows * per_row) return;
  const u64 r = i / per_row, j = (i % per_row) * 2;
  const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(in + (r * Lw + lo) * N + j);
  *reinterpret_cast<uint2*>(out + r * cnt * N + j) = make_uint2(static_cast<u32>(v.x), static_cast<u32>(v.y));
}

__global__ void k_limbs_to_u64(const u32* __restrict__ in, u64* __restrict__ out, u64 rows, u32 Lw, u32 lo, u32 cnt,
                               u32 N) {
  const u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
  const u64 per_row = static_cast<u64>(cnt) * N / 2;
  if (i >= rows * per_row) return;
  const u64 r = i / per_row, j = (i % per_row) * 2;
  const uint2 v = *reinterpret_cast<const uint2*>(in + r * cnt * N + j);
  *reinterpret_cast<ulonglong2*>(out + (r * Lw + lo) * N + j) = make_ulonglong2(v.x, v.y);
}

int launch_limbs_to_u32(const u64* in, u32* out, u64 rows, u32 Lw, u32 lo, u32 cnt, u32 N, cudaStream_t s) {
  const u64 threads = rows * cnt * N / 2;
  if (threads == 0) return 0;
  ProfScope ps_("k_limbs_to_u32", s);
  k_limbs_to_u32<<<(threads + 255) / 256, 256, 0, s>>>(in, out, rows, Lw, lo, cnt, N);
  return 1;
}

int launch_limbs_to_u64(const u32* in, u64* out, u64 rows, u32 Lw, u32 lo, u32 cnt, u32 N, cudaStream_t s) {
  const u64 threads = rows * cnt * N / 2;
  if (threads == 0) return 0;
  ProfScope ps_("k_limbs_to_u64", s);
  k_limbs_to_u64<<<(threads + 255) / 256, 256, 0, s>>>(in, out, rows, Lw, lo, cnt, N);
  return 1;
}

int launch_mac_conv_w(const MacConvArgsW& a, const BasisW& B, cudaStream_t s) {
  if (a.C * a.win * a.win > static_cast<u32>(kWMaxTaps) || a.N % 256 != 0) return -1;
  static const bool dw_on = [] {
    const char* e = getenv("HG_DWCONV");
    return !(e != nullptr && e[0] == '0');
  }();
  if (dw_on && a.groups > 1 && a.C == 1 && a.F == 1 && (a.win == 3 || a.win == 5) && a.groups <= 65535 &&
      a.polys * a.level <= 65535) {
    const size_t sm = static_cast<size_t>(a.IH) * a.IW * 32 * sizeof(ulonglong2);
    static const bool smem_on = [] {
      const char* e = getenv("HG_DWCONV_SMEM");
      return !(e != nullptr && e[0] == '0');
    }();
    if (smem_on && sm <= 112 * 1024 && a.N % 64 == 0) {  // input tile in shared memory
      auto k = a.win == 3 ? k_dwconv_ws<3> : k_dwconv_ws<5>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
      dim3 grid(a.N / 64, a.polys * a.level, a.groups);
      ProfScope ps_("k_dwconv_w", s);
      k<<<grid, 256, sm, s>>>(a, B);
      return 1;
    }
    dim3 grid(a.N / 256, a.polys * a.level, a.groups);
    ProfScope ps_("k_dwconv_w", s);
    if (a.win == 3)
      k_dwconv_w<3><<<grid, 128, 0, s>>>(a, B);
    else
      k_dwconv_w<5><<<grid, 128, 0, s>>>(a, B);
    return 1;
  }
  const u32 nchunks = (a.F + kWFT - 1) / kWFT;
  const u32 groups = a.groups ? a.groups : 1;
  if (static_cast<u64>(a.polys) * a.level * nchunks * groups > 65535) return -1;
  dim3 grid(a.N / 256, a.OH * a.OW, a.polys * a.level * nchunks * groups);
  { ProfScope ps_("k_mac_conv_w", s);
  k_mac_conv_w<<<grid, 128, 0, s>>>(a, B);
  }
  return 1;
}

int launch_elementwise_w(const EwArgsW& a, const BasisW& B, cudaStream_t s) {
  const u64 threads = a.count * a.polys_out * a.level * (a.N / 2);
  if (threads == 0) return 0;
  { ProfScope ps_("k_ew_w", s);
  k_ew_w<<<(threads + 255) / 256, 256, 0, s>>>(a, B);
  }
  return 1;
}

int launch_validate_w(const u64* w, u64 words, u32 level, u32 N, const BasisW& B, int* d_bad, cudaStream_t s) {
  if (words == 0) return 0;
  { ProfScope ps_("k_validate_w", s);
  k_validate_w<<<(words + 255) / 256, 256, 0, s>>>(w, words, level, N, B, d_bad);
  }
  return 1;
}

int launch_encode_scalars_w_f32(const float* vals, u64 count, u32 row_len, u32 row_stride, u64 limb_stride, u32 level,
                                double scale, u64* out, const BasisW& B, cudaStream_t s) {
  if (count == 0) return 0;
  { ProfScope ps_("k_encode_scalars_w", s);
  k_encode_scalars_w<float><<<(count + 127) / 128, 128, 0, s>>>(vals, count, row_len, row_stride, limb_stride, level,
                                                                scale, out, B);
  }
  return 1;
}

int launch_encode_scalars_w_f64(const double* vals, u64 count, u32 row_len, u32 row_stride, u64 limb_stride,
                                u32 level, double scale, u64* out, const BasisW& B, cudaStream_t s) {
  if (count == 0) return 0;
  { ProfScope ps_("k_encode_scalars_w", s);
  k_encode_scalars_w<double><<<(count + 127) / 128, 128, 0, s>>>(vals, count, row_len, row_stride, limb_stride, level,
                                                                 scale, out, B);
  }
  return 1;
}

}  // namespace hg

namespace hg {

__global__ void k_mags_to_residues_w(const ulonglong2* mags, u64 count_n, u32 n, u32 level, u32 lcount, u64* out,
                                     BasisW B) {
  const u64 idx = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= count_n) return;
  const ulonglong2 m = mags[idx];
  const bool neg = (m.y >> 63) != 0;
  const u64 hi = m.y & ~(1ull << 63);
  const u64 pt = idx / n, k = idx % n;
  for (u32 i = 0; i < lcount; ++i) {  // limbs [0, lcount)
    const DevPrimeW& P = B.p[i];
    u64 r = barrett128(m.x, hi, P);
    if (neg && r != 0) r = P.q - r;
    out[(pt * level + i) * n + k] = r;
  }
}

// encode's residues (the signed 128-bit magnitudes mod q, henet/encoding.hpp:160-168) fused
// into the plaintext NTT for the limbs below 2^30: each (plaintext, limb) CTA reduces its
// coefficients' magnitudes as it loads them (X mod q = (hi mod q)(2^64 mod q) + lo mod q) and
// writes only the NTT-domain residues -- no residue array round trip through HBM.
template <int LOGN>
__global__ void __launch_bounds__(1 << (LOGN - 5), (LOGN <= 13 ? 4 : HG_NTT14_MINB))
    k_pt_ntt_w32(const ulonglong2* mags, u64* out, u32 level, u32 lo, Basis B) {
  using NT = Ntt<LOGN, true>;
  extern __shared__ u32 sm32[];
  const u32 tid = threadIdx.x;
  const u32 cnt = level - lo;
  const u64 pt = blockIdx.x / cnt;
  const u32 limb = lo + blockIdx.x % cnt;
  const DevPrime& P = B.p[limb];
  const u32 t64 = mulmod(P.r32, P.r32, P);  // 2^64 mod q
  const ulonglong2* mg = mags + pt * NT::N;
  u32 x[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const ulonglong2 m = __ldg(&mg[NT::jA(tid, k)]);
    const bool neg = (m.y >> 63) != 0;
    const u32 r = addmod(reduce64(m.x, P), mulmod(reduce64(m.y & ~(1ull << 63), P), t64, P), P.q);
    x[k] = (neg && r != 0) ? P.q - r : r;
  }
  NT::forward(x, sm32, tid, P);
  u64* o = out + (pt * level + limb) * NT::N;
#pragma unroll
  for (int k = 0; k < 32; k += 4) {
    ulonglong2* d = reinterpret_cast<ulonglong2*>(o + NT::jC(tid, k));
    d[0] = make_ulonglong2(x[k], x[k + 1]);
    d[1] = make_ulonglong2(x[k + 2], x[k + 3]);
  }
}

int launch_pt_residues_ntt_w(int logn, const ulonglong2* mags, u64 count, u32 level, u64* out, const BasisW& B,
                             cudaStream_t s) {
  static const bool on = [] {
    const char* e = getenv("HG_ENCODE_FUSE");
    return !(e != nullptr && e[0] == '0');
  }();
  const u32 lo = wide_narrow_lo(B, level);
  if (!on || count == 0 || lo >= level) return -2;
  const u32 n = 1u << logn;
  int launches = 0;
  if (lo > 0) {  // the wide limbs: residues, then their u64 NTT
    const u64 total = count * n;
    {
      ProfScope ps_("k_mags_to_residues_w", s);
      k_mags_to_residues_w<<<(total + 255) / 256, 256, 0, s>>>(mags, total, n, level, lo, out, B);
    }
    ++launches;
  }
  HG_LOGN_SWITCH_W(logn, {
    if (lo > 0) {
      const size_t sm = sizeof(u64) * NttW<LN>::SMEM_WORDS;
      set_smem_w(k_ntt_w<LN, false>, sm);
      ProfScope ps_("k_ntt_w", s);
      k_ntt_w<LN, false><<<count * lo, 1 << (LN - 5), sm, s>>>(out, level, 0, lo, B);
      ++launches;
    }
    const size_t sm = sizeof(u32) * Ntt<LN, true>::SMEM_WORDS;
    set_smem_w(k_pt_ntt_w32<LN>, sm);
    ProfScope ps_("k_pt_ntt_w32", s);
    k_pt_ntt_w32<LN><<<count * (level - lo), 1 << (LN - 5), sm, s>>>(mags, out, level, lo,
                                                                     *static_cast<const Basis*>(B.narrow));
    ++launches;
  });
  return launches;
}

int launch_mags_to_residues_w(const ulonglong2* mags, u64 count, u32 n, u32 level, u64* out, const BasisW& B,
                              cudaStream_t s) {
  const u64 total = count * n;
  if (total == 0) return 0;
  { ProfScope ps_("k_mags_to_residues_w", s);
  k_mags_to_residues_w<<<(total + 255) / 256, 256, 0, s>>>(mags, total, n, level, level, out, B);
  }
  return 1;
}

}  // namespace hg
