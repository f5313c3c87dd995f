// SPDX-License-Identifier: Apache-2.0
//
// sm_100a kernels for the nGraph-HE2 encrypted-inference hot path.
//
//   k_ntt         batched per-limb negacyclic NTT / INTT       (henet/modmath.hpp:338-398)
//   k_rescale     NTT-domain rescale: INTT only the dropped limb, NTT the
//                 rounding correction under each kept prime   (henet/ckks.hpp:132-154, 504-519)
//   k_mac_dense   Dot: Y = W^T X per (poly, limb), lazy u64 accumulation,
//                 one Barrett reduction, bias in the epilogue  (henet/graph.hpp:905-954)
//   k_mac_conv    Convolution: implicit im2col, all filters of a position
//                 share the gathered inputs                   (henet/graph.hpp:956-993)
//   k_relin_*     square/tensor -> digit INTT -> key-switch inner product ->
//                 special-prime mod-down (+ fused rescale)    (henet/ckks.hpp:407-499)
//   k_ew          element-wise ct+ct, ct*pt, ct+pt, tensor    (henet/ckks.hpp:281-437)
//   k_encode_*    exact x87 scalar encoding and the FFT vector encoder
//                                                             (henet/encoding.hpp:122-197, fft.hpp)
#include <cuda_runtime.h>

#include <cstdio>

#include <cooperative_groups.h>

#include "hg_kernels.hpp"
#include "hg_x87.cuh"

namespace hg {

// ===========================================================================
// Batched NTT (hg_ntt_forward / hg_ntt_inverse)
// ===========================================================================
template <int LOGN, bool INV>
__global__ void __launch_bounds__(1 << (LOGN - 5), (LOGN <= 13 ? HG_NTT_TWS_MINB : 1)) k_ntt(u32* data, u32 level, Basis B) {
  using NT = Ntt<LOGN, true>;  // staged pass-B twiddles: 3 CTAs per SM
  extern __shared__ u32 sm[];
  const u32 tid = threadIdx.x;
  const u64 row = blockIdx.x;
  const DevPrime& P = B.p[row % level];
  u32* r = data + row * NT::N;
  u32 x[32];
  if (!INV) {
    NT::gload_A(x, r, tid);
    NT::forward(x, sm, tid, P);
    NT::gstore_C(x, r, tid);
  } else {
    NT::gload_C(x, r, tid);
    NT::inverse(x, sm, tid, P);
    NT::gstore_A(x, r, tid);
  }
}

// ===========================================================================
// Rescale (one CTA per (ciphertext, polynomial))
// ===========================================================================
// LAZY: the centred correction c (|c| <= q_{L-1}/2) enters each forward transform as
// c + pm_i < 4 q_i (the lazy transform's input range) instead of being reduced mod q_i.
// four consecutive residues of a u32 or u64 (WIO) row as a uint4
template <typename W>
__device__ __forceinline__ uint4 ld4(const W* p) {
  if constexpr (sizeof(W) == 4) {
    return __ldg(reinterpret_cast<const uint4*>(p));
  } else {
    const ulonglong2 a = __ldg(reinterpret_cast<const ulonglong2*>(p));
    const ulonglong2 b = __ldg(reinterpret_cast<const ulonglong2*>(p) + 1);
    return make_uint4(static_cast<u32>(a.x), static_cast<u32>(a.y), static_cast<u32>(b.x), static_cast<u32>(b.y));
  }
}
template <typename W>
__device__ __forceinline__ void st4(W* p, uint4 v) {
  if constexpr (sizeof(W) == 4) {
    *reinterpret_cast<uint4*>(p) = v;
  } else {
    reinterpret_cast<ulonglong2*>(p)[0] = make_ulonglong2(v.x, v.y);
    reinterpret_cast<ulonglong2*>(p)[1] = make_ulonglong2(v.z, v.w);
  }
}

// W = u64: the limbs are read and written in place in wide (u64) tensors (a.in64 / a.out64).
template <int LOGN, bool LAZY, typename W = u32>
__global__ void __launch_bounds__(1 << (LOGN - 5), (LOGN <= 13 ? HG_RESCALE_MINB : HG_NTT14_MINB)) k_rescale(RescaleArgs a, Basis B) {
  using NT = Ntt<LOGN, true>;  // staged pass-B twiddles: 3 CTAs per SM
  constexpr int N = NT::N;
  constexpr bool kWide = sizeof(W) == 8;
  extern __shared__ u32 sm[];
  const u32 tid = threadIdx.x;
  // rounding correction: thread-private row in tensor memory (cells [0, 32), i32 bits)
  TmemScratch<NT::T, HG_RESCALE_TMEM_CELLS> tm;
  tm.alloc(sm + NT::SMEM_WORDS, tid);
  const u64 row = blockIdx.x;
  const u32 L = a.level;
  const W* src;
  W* dst;
  if constexpr (kWide) {
    src = a.in64 + (row * a.io_level_in + a.io_off) * N;
    dst = a.out64 + (row * a.io_level_out + a.io_off) * N;
  } else {
    src = a.in + row * L * N;
    dst = a.out + row * (L - 1) * N;
  }

  u32 x[32];
  {
    const DevPrime& Pl = B.p[L - 1];
#pragma unroll
    for (int k = 0; k < 32; k += 4) {
      const uint4 v = ld4(src + static_cast<u64>(L - 1) * N + NT::jC(tid, k));
      x[k] = v.x;
      x[k + 1] = v.y;
      x[k + 2] = v.z;
      x[k + 3] = v.w;
    }
    NT::inverse(x, sm, tid, Pl);
#pragma unroll
    for (int c = 0; c < 32; c += 8) {
      u32 w[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) w[e] = static_cast<u32>(centered_round_rem(x[c + e], Pl));
      tm.st8(c, w);
    }
    decltype(tm)::wait_st();
  }
#pragma unroll 1
  for (u32 i = 0; i + 1 < L; ++i) {
    const DevPrime& Pi = B.p[i];
    const u32 pm = a.pm[i];
#pragma unroll
    for (int c = 0; c < 32; c += 8) {
      u32 v[8];
      tm.ld8(c, v);
      decltype(tm)::wait_ld();
#pragma unroll
      for (int e = 0; e < 8; ++e) x[c + e] = v[e] + pm;
    }
    if (!LAZY) {
#pragma unroll
      for (int k = 0; k < 32; ++k) x[k] = reduce32(x[k], Pi);
    }
    const W* in_i = src + static_cast<u64>(i) * N;
    W* out_i = dst + static_cast<u64>(i) * N;
    uint4 yv[8];  // issued before the transform so the loads overlap it
#pragma unroll
    for (int g = 0; g < 8; ++g) yv[g] = ld4(in_i + NT::jC(tid, 4 * g));
    NT::forward(x, sm, tid, Pi);
    const u32 q = Pi.q, pv = a.pinv[i], ps = a.pinv_sh[i];
#pragma unroll
    for (int k = 0; k < 32; k += 4) {
      const u32 j = NT::jC(tid, k);
      const uint4 y = yv[k >> 2];
      uint4 o;
      o.x = mul_shoup(y.x + q - x[k], pv, ps, q);
      o.y = mul_shoup(y.y + q - x[k + 1], pv, ps, q);
      o.z = mul_shoup(y.z + q - x[k + 2], pv, ps, q);
      o.w = mul_shoup(y.w + q - x[k + 3], pv, ps, q);
      st4(out_i + j, o);
    }
  }
  tm.free(tid);
}

// ===========================================================================
// Dense modular contraction (Dot)
//   grid.x = N / 128 coefficient tiles, grid.y = M tiles of 4*warps outputs,
//   grid.z = polys * level.  Warp w owns outputs m0 + 4w .. +4, lane owns
//   coefficients n0 + 4*lane .. +4 (16 u64 accumulators per thread, so up to
//   32 warps per CTA stay resident).  X and W tiles of BK = 16 taps are staged
//   in shared memory with cp.async (double buffered); every MAC is one
//   IMAD.WIDE.U32 into an un-reduced u64 lane, reduced once in the epilogue.
// ===========================================================================
constexpr int kBK = 16;
constexpr int kTM = 4;
constexpr int kBN = 128;
constexpr int kMaxWarps = 32;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int bytes = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// One BK-deep tile of the dense contraction; FOLD keeps 30-bit-limb accumulators
// below 2^64 by folding hi*2^32 into (2^32 mod q) every 8 taps.
template <bool FOLD>
__device__ __forceinline__ void mac_tile(u64 (&acc)[kTM][4], const u32 (*xs)[kBN], const u32 (*ws)[kTM * kMaxWarps],
                                         u32 lane, u32 warp, u64 r32) {
#pragma unroll
  for (int kk = 0; kk < kBK; ++kk) {
    const uint4 xv = *reinterpret_cast<const uint4*>(&xs[kk][lane * 4]);
    const uint4 wv = *reinterpret_cast<const uint4*>(&ws[kk][warp * kTM]);
    const u32 w[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
    for (int i = 0; i < kTM; ++i) {
      acc[i][0] += static_cast<u64>(w[i]) * xv.x;
      acc[i][1] += static_cast<u64>(w[i]) * xv.y;
      acc[i][2] += static_cast<u64>(w[i]) * xv.z;
      acc[i][3] += static_cast<u64>(w[i]) * xv.w;
    }
    if (FOLD && (kk & 7) == 7) {
#pragma unroll
      for (int i = 0; i < kTM; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = (acc[i][j] & 0xffffffffull) + (acc[i][j] >> 32) * r32;
    }
  }
}

constexpr int kStages = 4;
constexpr size_t kDenseSmem = static_cast<size_t>(kStages) * kBK * (kBN + kTM * kMaxWarps) * sizeof(u32);

__global__ void __launch_bounds__(kMaxWarps * 32, 1) k_mac_dense(MacDenseArgs a, Basis B) {
  extern __shared__ __align__(16) u32 dsm[];
  auto xs = reinterpret_cast<u32(*)[kBK][kBN]>(dsm);                                   // [kStages][kBK][kBN]
  auto ws = reinterpret_cast<u32(*)[kBK][kTM * kMaxWarps]>(dsm + kStages * kBK * kBN);  // [kStages][kBK][BM]
  const u32 warps = blockDim.x >> 5;
  const u32 BM = kTM * warps;
  const u32 tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const u32 n0 = blockIdx.x * kBN;
  const u32 m0 = blockIdx.y * BM;
  const u32 pl = blockIdx.z;  // poly * level + limb
  const u32 poly = pl / a.level, limb = pl % a.level;
  const DevPrime& P = B.p[limb];
  const u64 xstride = static_cast<u64>(a.polys) * a.x_level * a.N;  // words per input ct
  const u32* Xb = a.X + (static_cast<u64>(poly) * a.x_level + limb) * a.N + n0;
  const u32* Wb = a.W + static_cast<u64>(limb) * a.K * a.Mpad + m0;
  const bool fold = a.fold[limb] != 0;
  const u64 r32 = P.r32;

  const u32 ktiles = (a.K + kBK - 1) / kBK;
  auto load_tile = [&](u32 kt, int st) {
    for (u32 c = tid; c < kBK * (kBN / 4); c += blockDim.x) {
      const u32 r = c / (kBN / 4), col = (c % (kBN / 4)) * 4;
      const u32 k = kt * kBK + r;
      const bool v = k < a.K;
      cp_async16(&xs[st][r][col], Xb + (v ? static_cast<u64>(k) * xstride : 0) + col, v);
    }
    const u32 wq = BM / 4;
    for (u32 c = tid; c < kBK * wq; c += blockDim.x) {
      const u32 r = c / wq, col = (c % wq) * 4;
      const u32 k = kt * kBK + r;
      const bool v = k < a.K;
      cp_async16(&ws[st][r][col], Wb + (v ? static_cast<u64>(k) * a.Mpad : 0) + col, v);
    }
  };

  u64 acc[kTM][4];
#pragma unroll
  for (int i = 0; i < kTM; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0;

  // kStages-deep cp.async pipeline: tiles kt+1 .. kt+kStages-1 are in flight
  // while tile kt is multiplied.
#pragma unroll
  for (int st = 0; st < kStages - 1; ++st) {
    if (static_cast<u32>(st) < ktiles) load_tile(st, st);
    cp_async_commit();
  }
  for (u32 kt = 0; kt < ktiles; ++kt) {
    const int st = kt % kStages;
    cp_async_wait<kStages - 2>();
    __syncthreads();
    {
      const u32 nk = kt + kStages - 1;
      if (nk < ktiles) load_tile(nk, nk % kStages);
      cp_async_commit();
    }
    if (fold) {
      mac_tile<true>(acc, xs[st], ws[st], lane, warp, r32);
    } else {
      mac_tile<false>(acc, xs[st], ws[st], lane, warp, r32);
    }
  }

  const u32 q = P.q;
#pragma unroll
  for (int i = 0; i < kTM; ++i) {
    const u32 m = m0 + warp * kTM + i;
    if (m >= a.M) continue;
    u32 bv = 0;
    if (a.bias != nullptr && poly == 0) bv = __ldg(&a.bias[static_cast<u64>(limb) * a.Mpad + m]);
    uint4 o;
    o.x = addmod(reduce64(acc[i][0], P), bv, q);
    o.y = addmod(reduce64(acc[i][1], P), bv, q);
    o.z = addmod(reduce64(acc[i][2], P), bv, q);
    o.w = addmod(reduce64(acc[i][3], P), bv, q);
    u32* yp = a.Y + ((static_cast<u64>(m) * a.polys + poly) * a.level + limb) * a.N + n0 + lane * 4;
    *reinterpret_cast<uint4*>(yp) = o;
  }
}

// ===========================================================================
// Convolution (direct, implicit im2col)
//   grid.x = N / (4 * 256), grid.y = output positions, grid.z = polys * level *
//   filter chunks.  Each thread: 4 coefficients x FT filters; the gathered
//   input of the next tap is prefetched while the current tap is multiplied.
// ===========================================================================
#ifndef HG_CONV_PRE
#define HG_CONV_PRE 4  // gathered inputs in flight per thread: 0.401 ms per c2 step (3: 0.419; 5, 6: spills, 0.457 / 0.469)
#endif
constexpr int kMaxTaps = 1024;
constexpr int kConvThreads = 256;
#ifndef HG_CONV_PP
#define HG_CONV_PP 2
#endif
constexpr u32 kConvPos = HG_CONV_PP;  // output positions per CTA

// Tap loop of the convolution with its MACs split over two pipes: filters [0, KI) on
// IMAD.WIDE (fma pipe, u64 accumulators), filters [KI, FT) as DFMAs on the FP64 pipe.
// Exact: residues < 2^24-ish and at most 32 taps keep every partial sum an integer
// < 2^53 (host flag fp64[limb]); both accumulators are reduced the same way at the end.
// A u32 becomes a double with the 2^52 pair trick (MOV + DADD), not the slow I2F.F64
// (u32_to_f64, hg_device.cuh).

template <int FT>
struct ConvSplit {
  static constexpr int KI = (2 * FT + 2) / 5;  // IMAD.WIDE : DFMA issue-cycle balance (4 vs 2 + conversions)
  static constexpr int KF = FT - KI;
  static constexpr int KIP = (KI + 1) & ~1;    // per-tap weight rows padded for 64 / 128-bit loads
  static constexpr int KFP = (KF + 1) & ~1;
};

template <int FT, int kPre>
__device__ __forceinline__ void conv_taps_mixed(const MacConvArgs& a, const DevPrime& P, const uint2* tp,
                                                const u32* wmi, const double* wmd, u32 ntaps, const u32* Xb,
                                                u32 poly, u32 limb, u32 f0, u32 pos, u32 n) {
  constexpr int KI = ConvSplit<FT>::KI, KF = ConvSplit<FT>::KF;
  constexpr int KIP = ConvSplit<FT>::KIP, KFP = ConvSplit<FT>::KFP;
  u64 acc[KI > 0 ? KI : 1][4];
  double dacc[KF][4];
#pragma unroll
  for (int f = 0; f < KI; ++f)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[f][j] = 0;
#pragma unroll
  for (int f = 0; f < KF; ++f)
#pragma unroll
    for (int j = 0; j < 4; ++j) dacc[f][j] = 0.0;
  uint4 ring[kPre];
  u32 wring[kPre];
#pragma unroll
  for (int i = 0; i < kPre; ++i) {
    const uint2 e = static_cast<u32>(i) < ntaps ? __ldg(tp + i) : make_uint2(0, 0);
    wring[i] = e.y;
    ring[i] = (static_cast<u32>(i) < ntaps) ? __ldg(reinterpret_cast<const uint4*>(Xb + e.x))
                                            : make_uint4(0, 0, 0, 0);
  }
  for (u32 t0 = 0; t0 < ntaps; t0 += kPre) {
#pragma unroll
    for (int i = 0; i < kPre; ++i) {
      const u32 t = t0 + i;
      if (t >= ntaps) break;
      const uint4 xv = ring[i];
      u32 wi[KIP > 0 ? KIP : 2];
      double wf[KFP];
#pragma unroll
      for (int c = 0; c < KIP; c += 2) {
        const uint2 v = *reinterpret_cast<const uint2*>(wmi + wring[i] * KIP + c);
        wi[c] = v.x;
        wi[c + 1] = v.y;
      }
#pragma unroll
      for (int c = 0; c < KFP; c += 2) {
        const double2 v = *reinterpret_cast<const double2*>(wmd + wring[i] * KFP + c);
        wf[c] = v.x;
        wf[c + 1] = v.y;
      }
      if (t + kPre < ntaps) {
        const uint2 e = __ldg(tp + t + kPre);
        wring[i] = e.y;
        ring[i] = __ldg(reinterpret_cast<const uint4*>(Xb + e.x));
      }
#pragma unroll
      for (int f = 0; f < KI; ++f) {
        const u64 w = wi[f];
        acc[f][0] += w * xv.x;
        acc[f][1] += w * xv.y;
        acc[f][2] += w * xv.z;
        acc[f][3] += w * xv.w;
      }
      const double x0 = u32_to_f64(xv.x), x1 = u32_to_f64(xv.y), x2 = u32_to_f64(xv.z), x3 = u32_to_f64(xv.w);
#pragma unroll
      for (int f = 0; f < KF; ++f) {
        const double w = wf[f];
        dacc[f][0] = fma(w, x0, dacc[f][0]);
        dacc[f][1] = fma(w, x1, dacc[f][1]);
        dacc[f][2] = fma(w, x2, dacc[f][2]);
        dacc[f][3] = fma(w, x3, dacc[f][3]);
      }
    }
  }
  const u32 q = P.q;
#pragma unroll
  for (int f = 0; f < FT; ++f) {
    const u32 ff = f0 + f;
    if (ff >= a.F) continue;
    u32 bv = 0;
    if (a.bias != nullptr && poly == 0) bv = __ldg(&a.bias[static_cast<u64>(limb) * a.F + ff]);
    u64 v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j)
      v[j] = f < KI ? acc[f < KI ? f : 0][j] : static_cast<u64>(dacc[f < KI ? 0 : f - KI][j]);
    uint4 o;
    o.x = addmod(reduce64(v[0], P), bv, q);
    o.y = addmod(reduce64(v[1], P), bv, q);
    o.z = addmod(reduce64(v[2], P), bv, q);
    o.w = addmod(reduce64(v[3], P), bv, q);
    const u64 e = static_cast<u64>(ff) * a.OH * a.OW + pos;
    *reinterpret_cast<uint4*>(a.Y + ((e * a.polys + poly) * a.level + limb) * a.N + n) = o;
  }
}

template <int FT, int kPre>
__device__ __forceinline__ void conv_taps_int(const MacConvArgs& a, const DevPrime& P, const uint2* tp,
                                              const u32* wsm, u32 ntaps, const u32* Xb, u32 poly, u32 limb, u32 f0,
                                              u32 pos, u32 n) {
  const bool fold = a.fold[limb] != 0;
  const u64 r32 = P.r32;
  const u32 q = P.q;
  u64 acc[FT][4];
#pragma unroll
  for (int f = 0; f < FT; ++f)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[f][j] = 0;
  uint4 ring[kPre];
  u32 wring[kPre];
#pragma unroll
  for (int i = 0; i < kPre; ++i) {
    const uint2 e = static_cast<u32>(i) < ntaps ? __ldg(tp + i) : make_uint2(0, 0);
    wring[i] = e.y;
    ring[i] = (static_cast<u32>(i) < ntaps) ? __ldg(reinterpret_cast<const uint4*>(Xb + e.x))
                                            : make_uint4(0, 0, 0, 0);
  }
  for (u32 t0 = 0; t0 < ntaps; t0 += kPre) {
#pragma unroll
    for (int i = 0; i < kPre; ++i) {
      const u32 t = t0 + i;
      if (t >= ntaps) break;
      const uint4 xv = ring[i];
      const u32* wt = wsm + wring[i] * FT;
      if (t + kPre < ntaps) {
        const uint2 e = __ldg(tp + t + kPre);
        wring[i] = e.y;
        ring[i] = __ldg(reinterpret_cast<const uint4*>(Xb + e.x));
      }
#pragma unroll
      for (int f = 0; f < FT; ++f) {
        const u32 w = wt[f];
        acc[f][0] += static_cast<u64>(w) * xv.x;
        acc[f][1] += static_cast<u64>(w) * xv.y;
        acc[f][2] += static_cast<u64>(w) * xv.z;
        acc[f][3] += static_cast<u64>(w) * xv.w;
      }
      if (fold && (t & 7) == 7) {
#pragma unroll
        for (int f = 0; f < FT; ++f)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[f][j] = (acc[f][j] & 0xffffffffull) + (acc[f][j] >> 32) * r32;
      }
    }
  }
#pragma unroll
  for (int f = 0; f < FT; ++f) {
    const u32 ff = f0 + f;
    if (ff >= a.F) continue;
    u32 bv = 0;
    if (a.bias != nullptr && poly == 0) bv = __ldg(&a.bias[static_cast<u64>(limb) * a.F + ff]);
    uint4 o;
    o.x = addmod(reduce64(acc[f][0], P), bv, q);
    o.y = addmod(reduce64(acc[f][1], P), bv, q);
    o.z = addmod(reduce64(acc[f][2], P), bv, q);
    o.w = addmod(reduce64(acc[f][3], P), bv, q);
    const u64 e = static_cast<u64>(ff) * a.OH * a.OW + pos;
    *reinterpret_cast<uint4*>(a.Y + ((e * a.polys + poly) * a.level + limb) * a.N + n) = o;
  }
}

// CTA: kConvPos consecutive output positions x (4 * kConvThreads coefficients of one
// (poly, limb)) x FT filters.  The FT weights of every window tap are staged once
// ([window tap][FT]); each position's valid taps come from the host-built table.
template <int FT>
__global__ void __launch_bounds__(kConvThreads, 3) k_mac_conv(MacConvArgs a, Basis B) {
  __shared__ __align__(16) u32 wsm[kMaxTaps * FT];
  // the mixed path's (<= 32 taps) weights again, per tap: IMAD.WIDE filters as u32 pairs,
  // DFMA filters as pre-converted doubles (128-bit loads)
  __shared__ __align__(16) u32 wmi[32 * (ConvSplit<FT>::KIP > 0 ? ConvSplit<FT>::KIP : 2)];
  __shared__ __align__(16) double wmd[32 * ConvSplit<FT>::KFP];
  const u32 tid = threadIdx.x;
  const u32 npos = a.OH * a.OW;
  const u32 nchunks = (a.F + FT - 1) / FT;
  const u32 pl = blockIdx.z / nchunks;
  const u32 f0 = (blockIdx.z % nchunks) * FT;
  const u32 poly = pl / a.level, limb = pl % a.level;
  const DevPrime& P = B.p[limb];
  const u32 n = (blockIdx.x * blockDim.x + tid) * 4;
  const u32 taps_all = a.C * a.win * a.win;
  const u32* Wl = a.W + static_cast<u64>(limb) * a.F * taps_all;
  for (u32 i = tid; i < taps_all * FT; i += blockDim.x) {
    const u32 t = i / FT, f = i % FT;
    const u32 w = (f0 + f < a.F) ? __ldg(&Wl[static_cast<u64>(f0 + f) * taps_all + t]) : 0u;
    wsm[i] = w;
    if (t < 32) {
      constexpr int KI = ConvSplit<FT>::KI, KIP = ConvSplit<FT>::KIP, KFP = ConvSplit<FT>::KFP;
      if (static_cast<int>(f) < KI)
        wmi[t * KIP + f] = w;
      else
        wmd[t * KFP + (f - KI)] = static_cast<double>(w);
    }
  }
  if (tid < 32) {  // zero the padding slots
    constexpr int KI = ConvSplit<FT>::KI, KIP = ConvSplit<FT>::KIP, KF = ConvSplit<FT>::KF;
    constexpr int KFP = ConvSplit<FT>::KFP;
    for (int c = KI; c < KIP; ++c) wmi[tid * KIP + c] = 0u;
    for (int c = KF; c < KFP; ++c) wmd[tid * KFP + c] = 0.0;
  }
  __syncthreads();
  const u64 xstride = static_cast<u64>(a.polys) * a.x_level * a.N;
  const u32* Xb = a.X + (static_cast<u64>(poly) * a.x_level + limb) * a.N + n;
  const bool fp = a.fp64[limb] != 0;
  constexpr int kPre = HG_CONV_PRE;  // gathered inputs in flight
  const u32 p1 = min(npos, (blockIdx.y + 1) * kConvPos);
#pragma unroll 1
  for (u32 pos = blockIdx.y * kConvPos; pos < p1; ++pos) {
    // valid taps in ascending (c, ky, kx) order (henet/graph.hpp:976-989)
    const u32 off0 = __ldg(&a.tap_off[pos]);
    const u32 ntaps = __ldg(&a.tap_off[pos + 1]) - off0;
    if (fp && ntaps <= 32)
      conv_taps_mixed<FT, kPre>(a, P, a.taps + off0, wmi, wmd, ntaps, Xb, poly, limb, f0, pos, n);
    else
      conv_taps_int<FT, kPre>(a, P, a.taps + off0, wsm, ntaps, Xb, poly, limb, f0, pos, n);
  }
}

// ===========================================================================
// Relinearization (henet/ckks.hpp:442-499), three kernels:
//   K1 k_relin_digits  (ct, j):       c2_j -> INTT_j -> digit j (coefficient domain)
//   K2 k_relin_keysw   (ct, t<=level): sum_j NTT_t(digit_j mod q_t) * key[j][.][t];
//                                      t == level is the special prime P, whose
//                                      accumulators are INTT'd into the rounding
//                                      corrections of the mod-down.
//   K3 k_relin_moddown (ct, poly):    d + (acc - NTT(corr)) * P^-1 [+ rescale, with
//                                      both corrections merged into one NTT per limb]
// ===========================================================================
template <int LOGN, int MD>
__device__ __forceinline__ void load_c2(u32 (&y)[32], const RelinArgs& a, u64 ct, u32 j, const DevPrime& P,
                                        u32 tid) {
  using NT = Ntt<LOGN>;
  constexpr int N = NT::N;
  const u32 L = a.level;
  if (MD == 0) {
    NT::gload_C(y, a.A + ((ct * 3 + 2) * L + j) * N, tid);
  } else {
    u32 b1[32];
    NT::gload_C(y, a.A + ((ct * 2 + 1) * L + j) * N, tid);
    NT::gload_C(b1, a.Bm + ((ct * 2 + 1) * L + j) * N, tid);
#pragma unroll
    for (int k = 0; k < 32; ++k) y[k] = mulmod(y[k], b1[k], P);
  }
}

template <int LOGN, int MD>
__global__ void __launch_bounds__(1 << (LOGN - 5), (LOGN <= 13 ? HG_DIGITS_MINB : 1)) k_relin_digits(RelinArgs a, Basis B) {
  using NT = Ntt<LOGN, true>;  // staged pass-B twiddles: 3 CTAs per SM
  constexpr int N = NT::N;
  extern __shared__ u32 sm[];
  const u32 tid = threadIdx.x;
  const u64 ct = blockIdx.x / a.level;
  const u32 j = blockIdx.x % a.level;
  const DevPrime& P = B.p[j];
  u32 y[32];
  load_c2<LOGN, MD>(y, a, ct, j, P, tid);
  NT::inverse(y, sm, tid, P);
  NT::gstore_P(y, a.D + (ct * a.level + j) * N, tid);  // scratch: layout P
}

// SPECIAL: the CTAs of the special prime (grid = count), else limbs t < level
// (grid = count * level); split so neither body carries the other's code.
// The two accumulator rows live in tensor memory (TmemScratch: 64 cells per thread), so
// shared memory holds only the transform's exchange buffer and staged twiddles and
// 3 CTAs fit per SM.
template <int LOGN, int MD, bool SPECIAL>
__global__ void __launch_bounds__(1 << (LOGN - 5), (LOGN <= 13 ? HG_KEYSW_MINB : 1)) k_relin_keysw(RelinArgs a, Basis B) {
  using NT = Ntt<LOGN, true>;
  constexpr int N = NT::N;
  constexpr int T = NT::T;
  extern __shared__ u32 sm[];
  const u32 tid = threadIdx.x;
  TmemScratch<T> tm;
  tm.alloc(sm + NT::SMEM_WORDS, tid);
  // cells [0, 32): acc0 (c0 part), [32, 64): acc1, coefficient jC(tid, k) at cell k; values
  // kept in [0, 2q)
  const u32 L = a.level;
  const u64 ct = SPECIAL ? blockIdx.x : blockIdx.x / L;
  const u32 t = SPECIAL ? L : blockIdx.x % L;
  constexpr bool special = SPECIAL;
  const u32 bidx = special ? a.chain_len : t;  // basis index == key limb index
  const DevPrime& P = B.p[bidx];
  const u32 q = P.q, q2 = P.two_q;

  // acc{0,1} += y * key[j][{0,1}][t]
  auto mac = [&](const u32 (&y)[32], u32 j) {
    const u64 r0 = ((static_cast<u64>(j) * 2 + 0) * (a.chain_len + 1) + bidx) * N;
    const u64 r1 = ((static_cast<u64>(j) * 2 + 1) * (a.chain_len + 1) + bidx) * N;
    TmemScratch<T>::wait_st();  // the previous digit's stores of these cells
    if constexpr (kKeyShoup) {
      const uint2* k0 = static_cast<const uint2*>(a.key) + r0;
      const uint2* k1 = static_cast<const uint2*>(a.key) + r1;
      auto madd = [&](u32 acc, u32 x, u32 w, u32 wsh) { return csub(acc + mul_shoup_lazy(x, w, wsh, q), q2); };
      // key rows are L2-resident but far: issue a round of 4 pair-loads before using any
#pragma unroll
      for (int qr = 0; qr < 4; ++qr) {
        uint4 kv0[4], kv1[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const u32 jj = NT::jC(tid, qr * 8 + 2 * i);
          kv0[i] = __ldg(reinterpret_cast<const uint4*>(k0 + jj));
          kv1[i] = __ldg(reinterpret_cast<const uint4*>(k1 + jj));
        }
        u32 A0[8], A1[8];
        tm.ld8(qr * 8, A0);
        tm.ld8(32 + qr * 8, A1);
        TmemScratch<T>::wait_ld();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int k = qr * 8 + 2 * i;
          A0[2 * i] = madd(A0[2 * i], y[k], kv0[i].x, kv0[i].y);
          A0[2 * i + 1] = madd(A0[2 * i + 1], y[k + 1], kv0[i].z, kv0[i].w);
          A1[2 * i] = madd(A1[2 * i], y[k], kv1[i].x, kv1[i].y);
          A1[2 * i + 1] = madd(A1[2 * i + 1], y[k + 1], kv1[i].z, kv1[i].w);
        }
        tm.st8(qr * 8, A0);
        tm.st8(32 + qr * 8, A1);
      }
    } else {
      const u32* k0 = static_cast<const u32*>(a.key) + r0;
      const u32* k1 = static_cast<const u32*>(a.key) + r1;
      auto madd = [&](u32 acc, u32 x, u32 w) { return csub(acc + mulmod_lazy2(x, w, P), q2); };
#pragma unroll
      for (int qr = 0; qr < 4; ++qr) {
        uint4 kv0[2], kv1[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const u32 jj = NT::jC(tid, qr * 8 + 4 * h);
          kv0[h] = __ldg(reinterpret_cast<const uint4*>(k0 + jj));
          kv1[h] = __ldg(reinterpret_cast<const uint4*>(k1 + jj));
        }
        u32 A0[8], A1[8];
        tm.ld8(qr * 8, A0);
        tm.ld8(32 + qr * 8, A1);
        TmemScratch<T>::wait_ld();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int k = qr * 8 + 4 * h;
          A0[4 * h] = madd(A0[4 * h], y[k], kv0[h].x);
          A0[4 * h + 1] = madd(A0[4 * h + 1], y[k + 1], kv0[h].y);
          A0[4 * h + 2] = madd(A0[4 * h + 2], y[k + 2], kv0[h].z);
          A0[4 * h + 3] = madd(A0[4 * h + 3], y[k + 3], kv0[h].w);
          A1[4 * h] = madd(A1[4 * h], y[k], kv1[h].x);
          A1[4 * h + 1] = madd(A1[4 * h + 1], y[k + 1], kv1[h].y);
          A1[4 * h + 2] = madd(A1[4 * h + 2], y[k + 2], kv1[h].z);
          A1[4 * h + 3] = madd(A1[4 * h + 3], y[k + 3], kv1[h].w);
        }
        tm.st8(qr * 8, A0);
        tm.st8(32 + qr * 8, A1);
      }
    }
  };
  {
    const u32 z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int c = 0; c < 64; c += 8) tm.st8(c, z);
  }
  // Digits j != t (all j for the special prime): NTT_t(digit_j mod q_t), digit j+1
  // loaded during digit j's key products.  The loop body is branch-free: a j == t
  // test inside it makes ptxas duplicate the transform (instruction-cache misses).
  const u32 skip = special ? L : t;
  const u32 R = special ? L : L - 1;
#if HG_KEYSW_PREFETCH
  u32 nx[32];
  NT::gload_P(nx, a.D + (ct * L + (skip == 0 ? 1 : 0)) * N, tid);
#endif
  NT::stage_rowsB(P.fwdB, sm, tid);  // ordered before pass B by the transform's first barrier
#pragma unroll 1
  for (u32 r = 0; r < R; ++r) {
    const u32 j = r + (r >= skip ? 1 : 0);
    // digit mod q_t (henet/ckks.hpp:463): the lazy forward transform accepts inputs < 4 q_t
    // and returns canonical values, so only a digit of a prime >= 4 q_t needs reducing
    // (the 30-bit limb 0 under a 24-bit target).
    u32 y[32];
#if HG_KEYSW_PREFETCH
#pragma unroll
    for (int k = 0; k < 32; ++k) y[k] = nx[k];
#else
    // no register prefetch: the other resident CTAs cover the load (and no 32-register copy)
    NT::gload_P(y, a.D + (ct * L + j) * N, tid);
#endif
    // (the same test in the special-prime kernel: with P of the size of the largest chain
    // prime no digit needs reducing there)
    if ((B.p[j].q >> 2) >= q) {
#pragma unroll
      for (int k = 0; k < 32; ++k) y[k] = reduce32(y[k], P);
    }
    NT::forward(y, sm, tid, P, false);  // one prime per CTA: pass-B twiddles staged once, above
#if HG_KEYSW_PREFETCH
    const u32 jn = min(r + 1 + (r + 1 >= skip ? 1 : 0), L - 1);
    NT::gload_P(nx, a.D + (ct * L + jn) * N, tid);
#endif
    mac(y, j);
  }
  TmemScratch<T>::wait_st();
  if constexpr (!special) {
    // NTT_t(INTT_t(c2_t)) == c2_t: the digit's own limb needs no transform.
    u32 y[32];
    load_c2<LOGN, MD>(y, a, ct, t, P, tid);
    mac(y, t);
    TmemScratch<T>::wait_st();
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      u32* dst = a.ACC + ((ct * 2 + c) * L + t) * N;
#pragma unroll
      for (int k = 0; k < 32; k += 8) {
        u32 v[8];
        tm.ld8(c * 32 + k, v);
        TmemScratch<T>::wait_ld();
        *reinterpret_cast<uint4*>(dst + NT::jC(tid, k)) =
            make_uint4(csub(v[0], q), csub(v[1], q), csub(v[2], q), csub(v[3], q));
        *reinterpret_cast<uint4*>(dst + NT::jC(tid, k + 4)) =
            make_uint4(csub(v[4], q), csub(v[5], q), csub(v[6], q), csub(v[7], q));
      }
    }
  } else {
#pragma unroll 1
    for (int c = 0; c < 2; ++c) {
      u32 y[32];
#pragma unroll
      for (int k = 0; k < 32; k += 8) {
        u32 v[8];
        tm.ld8(c * 32 + k, v);
        TmemScratch<T>::wait_ld();
#pragma unroll
        for (int i = 0; i < 8; ++i) y[k + i] = csub(v[i], q);
      }
      NT::inverse(y, sm, tid, P);
      i32 cr[32];
#pragma unroll
      for (int k = 0; k < 32; ++k) cr[k] = centered_round_rem(y[k], P);
      NT::gstore_P(cr, a.CORR + (ct * 2 + c) * N, tid);  // scratch: layout P
    }
  }
  tm.free(tid);
}

// d0 = c0 (mode 0) or a0*b0; d1 = c1 (mode 0) or a0*b1 + a1*b0 (henet/ckks.hpp:407-437), four
// consecutive coefficients j..j+3 of limb i.
template <int MD>  // 0: three-poly input, 1: square (A == Bm), 2: product A x Bm
__device__ __forceinline__ uint4 load_d4(const RelinArgs& a, u64 ct, u32 poly, u32 i, u32 j, u32 N,
                                         const DevPrime& P) {
  const u32 L = a.level;
  auto ld = [&](const u32* base, u32 polys, u32 p) {
    return __ldg(reinterpret_cast<const uint4*>(base + ((ct * polys + p) * L + i) * static_cast<u64>(N) + j));
  };
  if (MD == 0) return ld(a.A, 3, poly);
  if (MD == 1) {
    // square (henet/ckks.hpp:424-437): d0 = c0^2, d1 = c0 c1 + c0 c1
    const uint4 x = ld(a.A, 2, 0), y = poly ? ld(a.A, 2, 1) : x;
    uint4 d = make_uint4(mulmod(x.x, y.x, P), mulmod(x.y, y.y, P), mulmod(x.z, y.z, P), mulmod(x.w, y.w, P));
    if (poly == 1) {
      d.x = addmod(d.x, d.x, P.q);
      d.y = addmod(d.y, d.y, P.q);
      d.z = addmod(d.z, d.z, P.q);
      d.w = addmod(d.w, d.w, P.q);
    }
    return d;
  }
  const uint4 x = ld(a.A, 2, 0), y = ld(a.Bm, 2, poly);
  uint4 d = make_uint4(mulmod(x.x, y.x, P), mulmod(x.y, y.y, P), mulmod(x.z, y.z, P), mulmod(x.w, y.w, P));
  if (poly == 1) {
    const uint4 u = ld(a.A, 2, 1), v = ld(a.Bm, 2, 0);
    d.x = addmod(d.x, mulmod(u.x, v.x, P), P.q);
    d.y = addmod(d.y, mulmod(u.y, v.y, P), P.q);
    d.z = addmod(d.z, mulmod(u.z, v.z, P), P.q);
    d.w = addmod(d.w, mulmod(u.w, v.w, P), P.q);
  }
  return d;
}

// MD selects the d0/d1 source (load_d4), RS whether the rescale is merged: one
// instantiation per combination keeps each kernel body inside the instruction cache.
template <int LOGN, int MD, bool RS>
__global__ void __launch_bounds__(1 << (LOGN - 5), (LOGN <= 13 ? (MD == 2 && HG_MODDOWN_MINB > 3 ? 3 : HG_MODDOWN_MINB) : 1))
    k_relin_moddown(RelinArgs a, Basis B) {  // MD == 2 (four input rows per limb) spills at 64 registers
  using NT = Ntt<LOGN, true>;
  constexpr int N = NT::N;
  constexpr int T = NT::T;
  extern __shared__ u32 sm[];
  const u32 tid = threadIdx.x;
  // special-prime (cps, cells [0, 32)) and rescale (crs, cells [32, 64)) corrections:
  // thread-private rows in tensor memory (see k_relin_keysw), i32 bit patterns
  TmemScratch<T> tm;
  tm.alloc(sm + NT::SMEM_WORDS, tid);
  const u32 L = a.level;
  const u64 ct = blockIdx.x >> 1;
  const u32 poly = blockIdx.x & 1;
  const u32 Lout = RS ? L - 1 : L;
  u32* dst = a.out + (ct * 2 + poly) * static_cast<u64>(Lout) * N;
  const u32* accp = a.ACC + (ct * 2 + poly) * static_cast<u64>(L) * N;
#pragma unroll
  for (int c = 0; c < 8; c += 2) {
    const int4* src = reinterpret_cast<const int4*>(a.CORR + (ct * 2 + poly) * N);  // layout P
    const int4 u = __ldg(src + c * T + tid), v = __ldg(src + (c + 1) * T + tid);
    const u32 w[8] = {static_cast<u32>(u.x), static_cast<u32>(u.y), static_cast<u32>(u.z), static_cast<u32>(u.w),
                      static_cast<u32>(v.x), static_cast<u32>(v.y), static_cast<u32>(v.z), static_cast<u32>(v.w)};
    tm.st8(4 * c, w);
  }
#if HG_MODDOWN_TOPINV
  if constexpr (RS) {
    // Top limb L-1 (dropped by the merged rescale): only its coefficient-domain value is
    // needed, for the rescale correction.  INTT is linear, so
    //   INTT(d + (acc - NTT(cps)) P^-1) = INTT(d + acc P^-1) - cps P^-1,
    // one inverse transform instead of a forward and an inverse one.
    const u32 i = L - 1;
    const DevPrime& Pi = B.p[i];
    const u32 q = Pi.q, pv = a.pinvP[i], ps = a.pinvP_sh[i], pm = a.pmP[i];
    u32 y[32];
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(accp + static_cast<u64>(i) * N + NT::jC(tid, 4 * g)));
      const uint4 d = load_d4<MD>(a, ct, poly, i, NT::jC(tid, 4 * g), N, Pi);
      // accP: acc * P^-1, canonical (the accumulators carry it already under kKeyPinv)
      auto accP = [&](u32 w) { return kKeyPinv ? w : mul_shoup(w, pv, ps, q); };
      y[4 * g] = addmod(d.x, accP(v.x), q);
      y[4 * g + 1] = addmod(d.y, accP(v.y), q);
      y[4 * g + 2] = addmod(d.z, accP(v.z), q);
      y[4 * g + 3] = addmod(d.w, accP(v.w), q);
    }
    NT::inverse(y, sm, tid, Pi);  // layout A, canonical: the layout of the cps cells
    TmemScratch<T>::wait_st();
#pragma unroll
    for (int c = 0; c < 32; c += 8) {
      u32 u[8], w[8];
      tm.ld8(c, u);
      TmemScratch<T>::wait_ld();
#pragma unroll
      for (int e = 0; e < 8; ++e)
        w[e] = static_cast<u32>(centered_round_rem(submod(y[c + e], mul_shoup(u[e] + pm, pv, ps, q), q), Pi));
      tm.st8(32 + c, w);
    }
  }
  constexpr bool kTopInLoop = false;
#else
  constexpr bool kTopInLoop = RS;
#endif
  // One loop, one inlined forward transform (the kernel body otherwise overflows the
  // instruction cache).  kTopInLoop (HG_MODDOWN_TOPINV=0): iteration 0 is the top limb
  // L-1, whose mod-down result feeds the rescale correction; iterations 1.. are limbs
  // 0..L-2.
#pragma unroll 1
  for (u32 it = (RS && !kTopInLoop) ? 1 : 0; it < L; ++it) {
    const bool top = kTopInLoop && (it == 0);
    const u32 i = RS ? (it == 0 ? L - 1 : it - 1) : it;
    const DevPrime& Pi = B.p[i];
    const u32 q = Pi.q, pv = a.pinvP[i], ps = a.pinvP_sh[i];
    // Transform inputs, lazily reduced (the forward transform takes values < 4q):
    //   rescale limbs: cps * P^-1 + crs = Shoup(cps + pm, P^-1) in [0, 2q) + (crs + q) in
    //   [0, 2q) (|crs| <= q_{L-1}/2 <= q, checked by the host);
    //   otherwise:     cps + pm reduced once (|cps| <= P/2 may exceed q).
    const u32 pm = a.pmP[i];
    u32 z[32];
    TmemScratch<T>::wait_st();  // the correction rows written before this limb
    if (RS && !top) {
#pragma unroll
      for (int c = 0; c < 32; c += 8) {
        u32 u[8], v[8];
        tm.ld8(c, u);
        tm.ld8(32 + c, v);
        TmemScratch<T>::wait_ld();
#pragma unroll
        for (int e = 0; e < 8; ++e) z[c + e] = mul_shoup_lazy(u[e] + pm, pv, ps, q) + (v[e] + q);
      }
    } else {
#pragma unroll
      for (int c = 0; c < 32; c += 8) {
        u32 u[8];
        tm.ld8(c, u);
        TmemScratch<T>::wait_ld();
        // kKeyPinv: the transform of cps * P^-1 (lazy, < 2q), to be subtracted from acc * P^-1
#pragma unroll
        for (int e = 0; e < 8; ++e)
          z[c + e] = kKeyPinv ? mul_shoup_lazy(u[e] + pm, pv, ps, q) : reduce32(u[e] + pm, Pi);
      }
    }
    // accumulator loads issued ahead of the transform; d products computed after it
#if HG_MODDOWN_PREFETCH
    uint4 vv[8];
#pragma unroll
    for (int g = 0; g < 8; ++g) vv[g] = __ldg(reinterpret_cast<const uint4*>(accp + static_cast<u64>(i) * N + NT::jC(tid, 4 * g)));
#define HG_MD_V(g) vv[g]
#else
#define HG_MD_V(g) __ldg(reinterpret_cast<const uint4*>(accp + static_cast<u64>(i) * N + NT::jC(tid, 4 * (g))))
#endif
    NT::forward(z, sm, tid, Pi);
    uint4 dd[8];
#pragma unroll
    for (int g = 0; g < 8; ++g) dd[g] = load_d4<MD>(a, ct, poly, i, NT::jC(tid, 4 * g), N, Pi);
    u32* out_i = dst + static_cast<u64>(i) * N;
    if (RS && !top) {
      const u32 lv = a.pinvL[i], ls = a.pinvL_sh[i];
#pragma unroll
      for (int k = 0; k < 32; k += 4) {
        const uint4 d = dd[k >> 2], v = HG_MD_V(k >> 2);
        uint4 o;
        // (d + acc * P^-1 - z) * q_{L-1}^-1 with a lazy inner product: < 4q + q, any u32
        // input is fine for the outer Shoup multiplication, which returns canonical
        auto accP = [&](u32 w) { return kKeyPinv ? w : mul_shoup_lazy(w, pv, ps, q); };
        o.x = mul_shoup(d.x + accP(v.x) + q - z[k], lv, ls, q);
        o.y = mul_shoup(d.y + accP(v.y) + q - z[k + 1], lv, ls, q);
        o.z = mul_shoup(d.z + accP(v.z) + q - z[k + 2], lv, ls, q);
        o.w = mul_shoup(d.w + accP(v.w) + q - z[k + 3], lv, ls, q);
        *reinterpret_cast<uint4*>(out_i + NT::jC(tid, k)) = o;
      }
    } else {
#pragma unroll
      for (int k = 0; k < 32; k += 4) {
        const uint4 d = dd[k >> 2], v = HG_MD_V(k >> 2);
        // d + (acc - NTT(cps)) P^-1; kKeyPinv: both terms carry P^-1 already, d + v + q - z < 3q
        auto fin = [&](u32 dd, u32 vv, u32 zz) {
          if (kKeyPinv) {
            const u32 r = dd + vv + q - zz;
            return csub(min(r, r - Pi.two_q), q);
          }
          return addmod(dd, mul_shoup(vv + q - zz, pv, ps, q), q);
        };
        z[k] = fin(d.x, v.x, z[k]);
        z[k + 1] = fin(d.y, v.y, z[k + 1]);
        z[k + 2] = fin(d.z, v.z, z[k + 2]);
        z[k + 3] = fin(d.w, v.w, z[k + 3]);
      }
      if (!RS) {
        NT::gstore_C(z, out_i, tid);
      } else {
        NT::inverse(z, sm, tid, Pi);
#pragma unroll
        for (int c = 0; c < 32; c += 8) {
          u32 w[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) w[e] = static_cast<u32>(centered_round_rem(z[c + e], Pi));
          tm.st8(32 + c, w);
        }
      }
    }
  }
  tm.free(tid);
}

// ===========================================================================
// Element-wise kernels.  One thread per 4 coefficients of one limb row.
// ===========================================================================
__global__ void k_ew(EwArgs a, Basis B) {
  const u32 N = a.N;
  const u64 rows = a.count * a.polys_out * a.level;
  const u64 tiles_per_row = N / 4;
  const u64 idx = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= rows * tiles_per_row) return;
  const u64 row = idx / tiles_per_row;
  const u32 n = static_cast<u32>(idx % tiles_per_row) * 4;
  const u32 limb = row % a.level;
  const u32 poly = (row / a.level) % a.polys_out;
  const u64 e = row / (static_cast<u64>(a.level) * a.polys_out);
  const DevPrime& P = B.p[limb];
  const u32 q = P.q;
  auto ld = [&](const u32* base, u32 polys, u32 p) {
    return *reinterpret_cast<const uint4*>(base + ((e * polys + p) * a.level + limb) * N + n);
  };
  uint4 o;
  switch (a.op) {
    case EwOp::AddCC: {
      const uint4 x = ld(a.a, a.polys_a, poly), y = ld(a.b, a.polys_a, poly);
      o = make_uint4(addmod(x.x, y.x, q), addmod(x.y, y.y, q), addmod(x.z, y.z, q), addmod(x.w, y.w, q));
      break;
    }
    case EwOp::MulScalar: {
      const uint4 x = ld(a.a, a.polys_a, poly);
      const u32 r = a.res[(a.per_element ? e / a.pt_div : 0) * a.level + limb];
      o = make_uint4(mulmod(x.x, r, P), mulmod(x.y, r, P), mulmod(x.z, r, P), mulmod(x.w, r, P));
      break;
    }
    case EwOp::AddScalar: {
      o = ld(a.a, a.polys_a, poly);
      if (poly == 0) {
        const u32 r = a.res[(a.per_element ? e / a.pt_div : 0) * a.level + limb];
        o = make_uint4(addmod(o.x, r, q), addmod(o.y, r, q), addmod(o.z, r, q), addmod(o.w, r, q));
      }
      break;
    }
    case EwOp::AddVector: {
      o = ld(a.a, a.polys_a, poly);
      if (poly == 0) {
        const uint4 y = *reinterpret_cast<const uint4*>(
            a.b + ((a.per_element ? e / a.pt_div : 0) * a.level + limb) * static_cast<u64>(N) + n);
        o = make_uint4(addmod(o.x, y.x, q), addmod(o.y, y.y, q), addmod(o.z, y.z, q), addmod(o.w, y.w, q));
      }
      break;
    }
    case EwOp::Tensor: {
      // out0 = a0 b0, out1 = a0 b1 + a1 b0, out2 = a1 b1
      uint4 x, y;
      if (poly == 0) { x = ld(a.a, 2, 0); y = ld(a.b, 2, 0); }
      else if (poly == 2) { x = ld(a.a, 2, 1); y = ld(a.b, 2, 1); }
      else { x = ld(a.a, 2, 0); y = ld(a.b, 2, 1); }
      o = make_uint4(mulmod(x.x, y.x, P), mulmod(x.y, y.y, P), mulmod(x.z, y.z, P), mulmod(x.w, y.w, P));
      if (poly == 1) {
        x = ld(a.a, 2, 1); y = ld(a.b, 2, 0);
        o.x = addmod(o.x, mulmod(x.x, y.x, P), q);
        o.y = addmod(o.y, mulmod(x.y, y.y, P), q);
        o.z = addmod(o.z, mulmod(x.z, y.z, P), q);
        o.w = addmod(o.w, mulmod(x.w, y.w, P), q);
      }
      break;
    }
    case EwOp::GatherMul: {
      const u32 src = a.gidx[e];
      if (src == 0xFFFFFFFFu) {
        o = make_uint4(0, 0, 0, 0);
      } else {
        const uint4 x = *reinterpret_cast<const uint4*>(a.a + ((static_cast<u64>(src) * a.polys_a + poly) * a.level + limb) * N + n);
        const u32 r = a.res[static_cast<u64>(a.gw[e]) * a.level + limb];
        o = make_uint4(mulmod(x.x, r, P), mulmod(x.y, r, P), mulmod(x.z, r, P), mulmod(x.w, r, P));
      }
      break;
    }
    case EwOp::Copy:
    default:
      o = ld(a.a, a.polys_a, poly);
      break;
  }
  *reinterpret_cast<uint4*>(a.out + ((e * a.polys_out + poly) * a.level + limb) * N + n) = o;
}

// ===========================================================================
// Host <-> device word conversion
// ===========================================================================
__global__ void k_narrow(const u64* in, u32* out, u64 words, u32 level, u32 N, Basis B, int* bad) {
  const u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= words) return;
  const u32 limb = (i / N) % level;
  const u64 w = in[i];
  if (w >= B.p[limb].q) atomicExch(bad, 1);
  out[i] = static_cast<u32>(w);
}

__global__ void k_widen(const u32* in, u64* out, u64 words) {
  const u64 i = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < words) out[i] = in[i];
}

// ===========================================================================
// Encoding.  x87 emulation: the reference computes
//   roundl((long double)value * (long double)scale)          (henet/encoding.hpp:122-126, 184)
// in 80-bit extended precision (64-bit mantissa, round-to-nearest-even),
// then rounds half away from zero.  The exact 106-bit product of the two
// double mantissas is rounded to 64 bits here the same way.
// ===========================================================================
template <typename T>
__global__ void k_encode_scalars(const T* vals, u64 count, u32 row_len, u32 row_stride, u64 limb_stride,
                                 u32 level, double scale, u32* out, Basis B) {
  const u64 v = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= count) return;
  const X87 x = x87_mul(static_cast<double>(vals[v]), scale);
  const unsigned __int128 mag = x87_roundl_mag(x);
  const u64 dst = (v / row_len) * row_stride + v % row_len;
  for (u32 i = 0; i < level; ++i) out[i * limb_stride + dst] = residue_mag(mag, x.neg, B.p[i]);
}

// Exact complex arithmetic in the order GCC emits for std::complex<double>
// without FMA: (a+bi)(c+di) = (ac - bd) + (ad + bc)i, every op rounded.
__device__ __forceinline__ double2 cmul_exact(double2 x, double2 w) {
  return make_double2(__dsub_rn(__dmul_rn(x.x, w.x), __dmul_rn(x.y, w.y)),
                      __dadd_rn(__dmul_rn(x.x, w.y), __dmul_rn(x.y, w.x)));
}

__device__ __forceinline__ u32 bitrev_n(u32 i, u32 logn) { return __brev(i) >> (32 - logn); }

// One CTA per plaintext; the FFT works on a global scratch row (L2 resident).
// SMEM: the n-point working array in shared memory (n <= 8192: 128 KB, one CTA per SM),
// else a global scratch row per plaintext (L2-resident).
template <bool SMEM>
__global__ void __launch_bounds__(1024) k_fft_encode(const double* slots, u32 n_slots, u32 n, u32 logn, u32 level,
                                                    double scale, const double2* roots, const double2* twist,
                                                    double2* scratch, ulonglong2* mags, unsigned long long* max_mant,
                                                    int* max_exp) {
  extern __shared__ double2 fft_sm[];
  const u64 pt = blockIdx.x;
  const u32 tid = threadIdx.x;
  double2* a = SMEM ? fft_sm : scratch + pt * n;
  const double2* rt = roots;
  if (SMEM) {  // the n/2 roots staged next to the working array
    double2* r = fft_sm + n;
    for (u32 i = tid; i < n / 2; i += blockDim.x) r[i] = roots[i];
    rt = r;
  }
  const double* s = slots + pt * 2 * static_cast<u64>(n_slots);
  // conjugate extension (henet/fft.hpp:59-63), then the bit-reversal permutation (:89-92):
  // element j lands at a[bitrev(j)] (coalesced slot reads)
  for (u32 j = tid; j < n; j += blockDim.x) {
    double2 e = make_double2(0.0, 0.0);
    if (j < n_slots) e = make_double2(s[2 * j], s[2 * j + 1]);
    else if (n - 1 - j < n_slots) { const u32 jj = n - 1 - j; e = make_double2(s[2 * jj], -s[2 * jj + 1]); }
    const u32 i = bitrev_n(j, logn);
    if (SMEM) a[i] = e; else __stcg(&a[i], e);
  }
  __syncthreads();
  // radix-2 DIT stages (henet/fft.hpp:93-104)
  for (u32 lh = 0; lh < logn; ++lh) {  // len = 2^(lh + 1), half = 2^lh (powers of two: shifts)
    const u32 half = 1u << lh, len = half << 1, step = n >> (lh + 1);
    for (u32 idx = tid; idx < n / 2; idx += blockDim.x) {
      const u32 base = (idx >> lh) << (lh + 1), k = idx & (half - 1);
      const double2 w = rt[k * step];
      const double2 u = SMEM ? a[base + k] : __ldcg(&a[base + k]);
      const double2 v = cmul_exact(SMEM ? a[base + k + half] : __ldcg(&a[base + k + half]), w);
      const double2 o0 = make_double2(__dadd_rn(u.x, v.x), __dadd_rn(u.y, v.y));
      const double2 o1 = make_double2(__dsub_rn(u.x, v.x), __dsub_rn(u.y, v.y));
      if (SMEM) {
        a[base + k] = o0;
        a[base + k + half] = o1;
      } else {
        __stcg(&a[base + k], o0);
        __stcg(&a[base + k + half], o1);
      }
    }
    __syncthreads();
  }
  // untwist, real part, 1/N (henet/fft.hpp:66-72), then x87 scale+round and residues
  // (henet/encoding.hpp:153-168)
  const double inv_n = 1.0 / static_cast<double>(n);
  __shared__ unsigned long long s_mant[512];
  __shared__ int s_exp[512];
  unsigned long long bm = 0;
  int be = -100000;
  for (u32 k = tid; k < n; k += blockDim.x) {
    const double2 e = SMEM ? a[k] : __ldcg(&a[k]);
    const double2 tw = twist[k];
    const double re = __dsub_rn(__dmul_rn(e.x, tw.x), __dmul_rn(e.y, -tw.y));
    const double coeff = __dmul_rn(re, inv_n);
    const X87 x = x87_mul(coeff, scale);
    if (x.mant != 0 && (x.exp > be || (x.exp == be && x.mant > bm))) { bm = x.mant; be = x.exp; }
    const unsigned __int128 mag = x87_roundl_mag(x);
    mags[pt * n + k] = make_ulonglong2(static_cast<u64>(mag), static_cast<u64>(mag >> 64) | (x.neg ? (1ull << 63) : 0));
  }
  // largest magnitude: warp shuffles, then one entry per warp
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long m2 = __shfl_xor_sync(0xffffffffu, bm, o);
    const int e2 = __shfl_xor_sync(0xffffffffu, be, o);
    if (m2 != 0 && (bm == 0 || e2 > be || (e2 == be && m2 > bm))) { bm = m2; be = e2; }
  }
  if ((tid & 31) == 0) {
    s_mant[tid >> 5] = bm;
    s_exp[tid >> 5] = be;
  }
  __syncthreads();
  if (tid == 0) {
    for (u32 t = 1; t < blockDim.x / 32; ++t) {
      if (s_mant[t] != 0 && (bm == 0 || s_exp[t] > be || (s_exp[t] == be && s_mant[t] > bm))) {
        bm = s_mant[t];
        be = s_exp[t];
      }
    }
    max_mant[pt] = bm;
    max_exp[pt] = be;
  }
}

// n = 2^14 (the BASELINE c4 ring): the 256 KB working array does not fit one CTA's shared
// memory, so a 2-CTA cluster splits it: CTA r holds positions [r n/2, (r+1) n/2) and runs the
// first log2(n) - 1 stages locally (a block of len <= n/2 never crosses the halves); the last
// stage pairs (k, k + n/2) across the cluster through distributed shared memory.  Same
// butterflies, twiddles and roundings as k_fft_encode, so the same bits.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(1024)
    k_fft_encode2(const double* slots, u32 n_slots, u32 n, u32 logn, u32 level, double scale, const double2* roots,
                  const double2* twist, ulonglong2* mags, unsigned long long* max_mant, int* max_exp) {
  extern __shared__ double2 f2_sm[];
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const u32 r = cluster.block_rank();
  const u64 pt = blockIdx.x >> 1;
  const u32 tid = threadIdx.x, HN = n >> 1;
  double2* a = f2_sm;
  const double* s = slots + pt * 2 * static_cast<u64>(n_slots);
  for (u32 ii = tid; ii < HN; ii += blockDim.x) {  // position i = r HN + ii holds element bitrev(i)
    const u32 j = bitrev_n(r * HN + ii, logn);
    double2 e = make_double2(0.0, 0.0);
    if (j < n_slots) e = make_double2(s[2 * j], s[2 * j + 1]);
    else if (n - 1 - j < n_slots) { const u32 jj = n - 1 - j; e = make_double2(s[2 * jj], -s[2 * jj + 1]); }
    a[ii] = e;
  }
  __syncthreads();
  for (u32 lh = 0; lh + 1 < logn; ++lh) {
    const u32 half = 1u << lh, step = n >> (lh + 1);
    for (u32 idx = tid; idx < HN / 2; idx += blockDim.x) {
      const u32 base = (idx >> lh) << (lh + 1), k = idx & (half - 1);
      const double2 w = __ldg(&roots[k * step]);
      const double2 u = a[base + k];
      const double2 v = cmul_exact(a[base + k + half], w);
      a[base + k] = make_double2(__dadd_rn(u.x, v.x), __dadd_rn(u.y, v.y));
      a[base + k + half] = make_double2(__dsub_rn(u.x, v.x), __dsub_rn(u.y, v.y));
    }
    __syncthreads();
  }
  cluster.sync();
  {
    double2* h0 = cluster.map_shared_rank(a, 0);
    double2* h1 = cluster.map_shared_rank(a, 1);
    for (u32 kk = tid; kk < HN / 2; kk += blockDim.x) {  // last stage: step 1, pairs (k, k + HN)
      const u32 k = r * (HN / 2) + kk;
      const double2 w = __ldg(&roots[k]);
      const double2 u = h0[k];
      const double2 v = cmul_exact(h1[k], w);
      h0[k] = make_double2(__dadd_rn(u.x, v.x), __dadd_rn(u.y, v.y));
      h1[k] = make_double2(__dsub_rn(u.x, v.x), __dsub_rn(u.y, v.y));
    }
  }
  cluster.sync();
  const double inv_n = 1.0 / static_cast<double>(n);
  __shared__ unsigned long long s_mant[32];
  __shared__ int s_exp[32];
  unsigned long long bm = 0;
  int be = -100000;
  for (u32 kk = tid; kk < HN; kk += blockDim.x) {
    const u32 k = r * HN + kk;
    const double2 e = a[kk];
    const double2 tw = twist[k];
    const double re = __dsub_rn(__dmul_rn(e.x, tw.x), __dmul_rn(e.y, -tw.y));
    const double coeff = __dmul_rn(re, inv_n);
    const X87 x = x87_mul(coeff, scale);
    if (x.mant != 0 && (x.exp > be || (x.exp == be && x.mant > bm))) { bm = x.mant; be = x.exp; }
    const unsigned __int128 mag = x87_roundl_mag(x);
    mags[pt * n + k] = make_ulonglong2(static_cast<u64>(mag), static_cast<u64>(mag >> 64) | (x.neg ? (1ull << 63) : 0));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long m2 = __shfl_xor_sync(0xffffffffu, bm, o);
    const int e2 = __shfl_xor_sync(0xffffffffu, be, o);
    if (m2 != 0 && (bm == 0 || e2 > be || (e2 == be && m2 > bm))) { bm = m2; be = e2; }
  }
  if ((tid & 31) == 0) {
    s_mant[tid >> 5] = bm;
    s_exp[tid >> 5] = be;
  }
  __syncthreads();
  if (tid == 0) {
    for (u32 t = 1; t < blockDim.x / 32; ++t) {
      if (s_mant[t] != 0 && (bm == 0 || s_exp[t] > be || (s_exp[t] == be && s_mant[t] > bm))) {
        bm = s_mant[t];
        be = s_exp[t];
      }
    }
    s_mant[0] = bm;
    s_exp[0] = be;
  }
  cluster.sync();  // both halves' maxima published
  if (r == 0 && tid == 0) {
    const unsigned long long m2 = *cluster.map_shared_rank(&s_mant[0], 1);
    const int e2 = *cluster.map_shared_rank(&s_exp[0], 1);
    if (m2 != 0 && (bm == 0 || e2 > be || (e2 == be && m2 > bm))) { bm = m2; be = e2; }
    max_mant[pt] = bm;
    max_exp[pt] = be;
  }
  cluster.sync();  // the peer's shared memory outlives the read above
}

// Signed 128-bit magnitudes -> residues per limb (coefficient domain), u32 basis.
__global__ void k_mags_to_residues(const ulonglong2* mags, u64 count_n, u32 n, u32 level, u32* out, Basis B) {
  const u64 idx = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= count_n) return;
  const ulonglong2 m = mags[idx];
  const bool neg = (m.y >> 63) != 0;
  const unsigned __int128 mag = (static_cast<unsigned __int128>(m.y & ~(1ull << 63)) << 64) | m.x;
  const u64 pt = idx / n, k = idx % n;
  for (u32 i = 0; i < level; ++i) out[(pt * level + i) * n + k] = residue_mag(mag, neg, B.p[i]);
}

// ===========================================================================
// IMAD.WIDE throughput probe (register only)
// ===========================================================================
template <int KIND>
__global__ void k_imad_probe(u64* sink, u32 iters, u32 seed) {
  // KIND 0: IMAD (mad.lo.u32), 1: IMAD.WIDE (mul.wide.u32, high word consumed), 2: IMAD.HI (mul.hi.u32),
  // 3: Shoup lazy modular product (IMAD.HI + 2 IMAD; IMAD.HI/IMAD.WIDE issue at a
  //    quarter of the FFMA rate on sm_100, IMAD at half, so this is the NTT's unit)
  u32 a[8];
  u64 c[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { a[i] = (threadIdx.x ^ seed) * (2 * i + 3) + i; c[i] = i; }
  u32 b = seed | 1;
  for (u32 it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (KIND == 1) {
          // dependent chain x <- hi(x * b): a loop-invariant `c += a*b` would be strength-
          // reduced by ptxas into 64-bit adds and measure IADD3, not IMAD.WIDE
          u64 p;
          asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(static_cast<u32>(c[i]) ^ a[i]), "r"(b));
          c[i] = p >> 32;
        } else if (KIND == 0) {
          u32 lo = static_cast<u32>(c[i]);
          asm volatile("mad.lo.u32 %0, %1, %2, %0;" : "+r"(lo) : "r"(a[i]), "r"(b));
          c[i] = lo;
        } else if (KIND == 2) {
          u32 lo = static_cast<u32>(c[i]);
          asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(lo) : "r"(a[i] ^ lo), "r"(b));
          c[i] = lo;
        } else {  // KIND 3: Shoup lazy product chain x <- x*w - hi(x*wsh)*q (IMAD.HI + 2 IMAD)
          u32 x = static_cast<u32>(c[i]), h, lo;
          asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(h) : "r"(x), "r"(a[i]));
          asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(lo) : "r"(x), "r"(b));
          asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(x) : "r"(h), "r"(0xc0004001u), "r"(lo));
          c[i] = x;
        }
      }
    }
    b += 2;
  }
  u64 s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= c[i];
  if (s == 0x12345) sink[0] = s;
}

// ===========================================================================
// Per-kernel CUDA-event profiler (off by default; bench.py turns it on for its
// roofline pass).  Events are recorded on the launch stream around each kernel.
// ===========================================================================
}  // namespace hg
#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <vector>
namespace hg {
namespace {
struct ProfRec {
  const char* name;
  cudaEvent_t e0, e1;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<ProfRec> g_prof;
}  // namespace

static std::atomic<u64> g_launches{0};
u64 launches_total() { return g_launches.load(std::memory_order_relaxed); }

ProfScope::ProfScope(const char* n, cudaStream_t st) : name(n), s(st) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  if (!g_prof_on) return;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
}

ProfScope::~ProfScope() {
  if (!e0) return;
  cudaEventRecord(e1, s);
  std::lock_guard<std::mutex> g(g_prof_mu);
  g_prof.push_back({name, e0, e1});
}

void prof_enable(bool on) { g_prof_on = on; }

std::string prof_report() {
  std::lock_guard<std::mutex> g(g_prof_mu);
  std::map<std::string, std::pair<double, int>> agg;
  for (auto& r : g_prof) {
    cudaEventSynchronize(r.e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, r.e0, r.e1);
    auto& a = agg[r.name];
    a.first += ms;
    a.second += 1;
    cudaEventDestroy(r.e0);
    cudaEventDestroy(r.e1);
  }
  g_prof.clear();
  std::string out = "{";
  bool first = true;
  for (auto& kv : agg) {
    char buf[256];
    snprintf(buf, sizeof(buf), "%s\"%s\": {\"ms\": %.6f, \"launches\": %d}", first ? "" : ", ", kv.first.c_str(),
             kv.second.first, kv.second.second);
    out += buf;
    first = false;
  }
  return out + "}";
}

// ===========================================================================
// Launchers
// ===========================================================================
#define HG_LOGN_SWITCH(logn, ...)                   \
  switch (logn) {                                    \
    case 12: { constexpr int LN = 12; __VA_ARGS__; } break; \
    case 13: { constexpr int LN = 13; __VA_ARGS__; } break; \
    case 14: { constexpr int LN = 14; __VA_ARGS__; } break; \
    default: return -1;                              \
  }

template <typename K>
static void set_smem(K kernel, size_t bytes) {
  if (bytes > 48 * 1024) cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
}

int launch_ntt(int logn, u32* data, u64 rows, u32 level, bool inverse, const Basis& B, cudaStream_t s) {
  if (rows == 0) return 0;
  HG_LOGN_SWITCH(logn, {
    const size_t sm = sizeof(u32) * Ntt<LN, true>::SMEM_WORDS;
    if (inverse) {
      set_smem(k_ntt<LN, true>, sm);
      ProfScope ps("k_intt", s);
      k_ntt<LN, true><<<rows, 1 << (LN - 5), sm, s>>>(data, level, B);
    } else {
      set_smem(k_ntt<LN, false>, sm);
      ProfScope ps("k_ntt", s);
      k_ntt<LN, false><<<rows, 1 << (LN - 5), sm, s>>>(data, level, B);
    }
  });
  return 1;
}

int launch_rescale(int logn, const RescaleArgs& a, const Basis& B, cudaStream_t s) {
  if (a.rows == 0) return 0;
  HG_LOGN_SWITCH(logn, {
    const size_t sm = sizeof(u32) * (Ntt<LN, true>::SMEM_WORDS + 4);
    auto rk = a.in64 != nullptr ? (a.lazy ? k_rescale<LN, true, u64> : k_rescale<LN, false, u64>)
                                : (a.lazy ? k_rescale<LN, true> : k_rescale<LN, false>);
    set_smem(rk, sm);
    ProfScope ps("k_rescale", s);
    rk<<<a.rows, 1 << (LN - 5), sm, s>>>(a, B);
  });
  return 1;
}

u32 mac_dense_warps(u32 M) { return std::min<u32>(kMaxWarps, (M + kTM - 1) / kTM); }

int launch_mac_dense(const MacDenseArgs& a, const Basis& B, cudaStream_t s) {
  const u32 warps = mac_dense_warps(a.M);
  const u32 BM = warps * kTM;
  if (a.Mpad % BM != 0 || a.N % kBN != 0) return -1;
  dim3 grid(a.N / kBN, (a.M + BM - 1) / BM, a.polys * a.level);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_mac_dense, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kDenseSmem));
    attr = true;
  }
  ProfScope ps("k_mac_dense", s);
  k_mac_dense<<<grid, warps * 32, kDenseSmem, s>>>(a, B);
  return 1;
}

template <int FT>
static void conv_launch(const MacConvArgs& a, const Basis& B, cudaStream_t s) {
  const u32 nchunks = (a.F + FT - 1) / FT;
  dim3 grid(a.N / (4 * kConvThreads), (a.OH * a.OW + kConvPos - 1) / kConvPos, a.polys * a.level * nchunks);
  ProfScope ps("k_mac_conv", s);
  k_mac_conv<FT><<<grid, kConvThreads, 0, s>>>(a, B);
}

int launch_mac_conv(const MacConvArgs& a, const Basis& B, cudaStream_t s) {
  if (a.C * a.win * a.win > static_cast<u32>(kMaxTaps) || a.N % (4 * kConvThreads) != 0) return -1;
  switch (a.F) {
    case 1: conv_launch<1>(a, B, s); break;
    case 2: conv_launch<2>(a, B, s); break;
    case 3: conv_launch<3>(a, B, s); break;
    case 4: conv_launch<4>(a, B, s); break;
    case 5: conv_launch<5>(a, B, s); break;
    case 6: conv_launch<6>(a, B, s); break;
    case 7: conv_launch<7>(a, B, s); break;
    default: conv_launch<8>(a, B, s); break;
  }
  return 1;
}

// One non-blocking auxiliary stream per device for intra-op fork/join (HG_AUX_STREAM=0 off).
static cudaStream_t aux_stream(int idx = 0) {
  static const bool on = [] {
    const char* e = getenv("HG_AUX_STREAM");
    return !(e != nullptr && e[0] == '0');
  }();
  if (!on || g_prof_on) return nullptr;  // the per-kernel profiler serialises launches for attribution
  static std::mutex mu;
  static cudaStream_t streams[64][3] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64 || idx < 0 || idx >= 3) return nullptr;
  std::lock_guard<std::mutex> g(mu);
  if (!streams[dev][idx]) cudaStreamCreateWithFlags(&streams[dev][idx], cudaStreamNonBlocking);
  return streams[dev][idx];
}

#ifndef HG_RELIN_SPECIAL_STREAMS
#define HG_RELIN_SPECIAL_STREAMS 0
#endif
// One relinearisation chain (digits -> special + limb key switches -> mod-down) on stream
// s; the special-prime key switch runs on `ss` (== s, or an auxiliary stream it forks to).
template <int LN>
static void relin_chain(const RelinArgs& a, const Basis& B, cudaStream_t s, cudaStream_t aux_special) {
  const size_t sm1 = sizeof(u32) * Ntt<LN, true>::SMEM_WORDS;         // digits (staged twiddles)
  const size_t smk = sizeof(u32) * (Ntt<LN, true>::SMEM_WORDS + 4);  // key switch, mod-down
  const int T = 1 << (LN - 5);
  const bool prod = a.mode != 0;
  auto dk = prod ? k_relin_digits<LN, 1> : k_relin_digits<LN, 0>;
  auto kn = prod ? k_relin_keysw<LN, 1, false> : k_relin_keysw<LN, 0, false>;
  auto ks = prod ? k_relin_keysw<LN, 1, true> : k_relin_keysw<LN, 0, true>;
  set_smem(dk, sm1);
  set_smem(kn, smk);
  set_smem(ks, smk);
  { ProfScope ps("k_relin_digits", s);
  dk<<<a.count * a.level, T, sm1, s>>>(a, B);
  }
  cudaEvent_t fork = nullptr, join = nullptr;
  if (aux_special) {
    cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&join, cudaEventDisableTiming);
    cudaEventRecord(fork, s);
    cudaStreamWaitEvent(aux_special, fork, 0);
  }
  const cudaStream_t ss = aux_special ? aux_special : s;
  { ProfScope ps("k_relin_keysw", ss);
  ks<<<a.count, T, smk, ss>>>(a, B);
  }
  { ProfScope ps("k_relin_keysw", s);
  kn<<<a.count * a.level, T, smk, s>>>(a, B);
  }
  if (aux_special) {
    cudaEventRecord(join, aux_special);
    cudaStreamWaitEvent(s, join, 0);
    cudaEventDestroy(fork);
    cudaEventDestroy(join);
  }
  { ProfScope ps("k_relin_moddown", s);
  const int md = a.mode == 0 ? 0 : (a.A == a.Bm ? 1 : 2);
  auto mdk = md == 0 ? (a.rescale ? k_relin_moddown<LN, 0, true> : k_relin_moddown<LN, 0, false>)
           : md == 1 ? (a.rescale ? k_relin_moddown<LN, 1, true> : k_relin_moddown<LN, 1, false>)
                     : (a.rescale ? k_relin_moddown<LN, 2, true> : k_relin_moddown<LN, 2, false>);
  set_smem(mdk, smk);
  mdk<<<a.count * 2, T, smk, s>>>(a, B);
  }
}

int launch_relin(int logn, const RelinArgs& a, const Basis& B, cudaStream_t s) {
  if (a.count == 0) return 0;
  // Large batches run as two halves on two streams: one half's key switch (L1-bound) then
  // shares SMs with the other half's mod-down (ALU/FMA-bound).  Small batches keep one chain,
  // with the special-prime key switch on the auxiliary stream (its `count` CTAs alone would
  // leave most SMs idle).
  static const u64 split_min = [] {
    const char* e = getenv("HG_RELIN_SPLIT_MIN");
    return e ? static_cast<u64>(atoll(e)) : 256ull;
  }();
  cudaStream_t aux = aux_stream();
  HG_LOGN_SWITCH(logn, {
    const u64 N = 1ull << LN, L = a.level, Lout = a.rescale ? L - 1 : L;
    if (aux && split_min > 0 && a.count >= split_min) {
      const u64 n0 = a.count / 2;
      RelinArgs h0 = a, h1 = a;
      h0.count = n0;
      h1.count = a.count - n0;
      const u64 in_polys = a.mode == 0 ? 3 : 2;
      h1.A = a.A + n0 * in_polys * L * N;
      h1.Bm = a.Bm == a.A ? h1.A : a.Bm + n0 * 2 * L * N;
      h1.D = a.D + n0 * L * N;
      h1.ACC = a.ACC + n0 * 2 * L * N;
      h1.CORR = a.CORR + n0 * 2 * N;
      h1.out = a.out + n0 * 2 * Lout * N;
      cudaEvent_t fork, join;
      cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
      cudaEventCreateWithFlags(&join, cudaEventDisableTiming);
      cudaEventRecord(fork, s);
      cudaStreamWaitEvent(aux, fork, 0);
#if HG_RELIN_SPECIAL_STREAMS
      // each half's special-prime key switch (count CTAs: under three per SM) beside its limb kernel
      relin_chain<LN>(h0, B, s, aux_stream(1));
      relin_chain<LN>(h1, B, aux, aux_stream(2));
#else
      relin_chain<LN>(h0, B, s, nullptr);
      relin_chain<LN>(h1, B, aux, nullptr);
#endif
      cudaEventRecord(join, aux);
      cudaStreamWaitEvent(s, join, 0);
      cudaEventDestroy(fork);
      cudaEventDestroy(join);
    } else {
      relin_chain<LN>(a, B, s, aux);
    }
  });
  return 3;
}

int launch_elementwise(const EwArgs& a, const Basis& B, cudaStream_t s) {
  const u64 threads = a.count * a.polys_out * a.level * (a.N / 4);
  if (threads == 0) return 0;
  ProfScope ps("k_ew", s);
  k_ew<<<(threads + 255) / 256, 256, 0, s>>>(a, B);
  return 1;
}

int launch_narrow(const u64* in, u32* out, u64 words, u32 level, u32 N, const Basis& B, int* d_bad,
                  cudaStream_t s) {
  if (words == 0) return 0;
  ProfScope ps("k_narrow", s);
  k_narrow<<<(words + 255) / 256, 256, 0, s>>>(in, out, words, level, N, B, d_bad);
  return 1;
}

int launch_widen(const u32* in, u64* out, u64 words, cudaStream_t s) {
  if (words == 0) return 0;
  ProfScope ps("k_widen", s);
  k_widen<<<(words + 255) / 256, 256, 0, s>>>(in, out, words);
  return 1;
}

int launch_encode_scalars_f32(const float* vals, u64 count, u32 row_len, u32 row_stride, u64 limb_stride,
                              u32 level, double scale, u32* out, const Basis& B, cudaStream_t s) {
  if (count == 0) return 0;
  ProfScope ps("k_encode_scalars", s);
  k_encode_scalars<float><<<(count + 127) / 128, 128, 0, s>>>(vals, count, row_len, row_stride, limb_stride,
                                                              level, scale, out, B);
  return 1;
}

int launch_encode_scalars_f64(const double* vals, u64 count, u32 row_len, u32 row_stride, u64 limb_stride,
                              u32 level, double scale, u32* out, const Basis& B, cudaStream_t s) {
  if (count == 0) return 0;
  ProfScope ps("k_encode_scalars", s);
  k_encode_scalars<double><<<(count + 127) / 128, 128, 0, s>>>(vals, count, row_len, row_stride, limb_stride,
                                                               level, scale, out, B);
  return 1;
}

// HG_FFT_CLUSTER=0: the n = 2^14 FFTs on the single-CTA global-memory kernels
bool fft_cluster_on() {
  static const bool on = [] {
    const char* e = getenv("HG_FFT_CLUSTER");
    return !(e != nullptr && e[0] == '0');
  }();
  return on;
}

int launch_fft_encode(const double* slots, u32 n_slots, u64 count, u32 n, u32 level, double scale,
                      const double2* roots, const double2* twist, double2* scratch, ulonglong2* mags,
                      unsigned long long* max_mant, int* max_exp, cudaStream_t s) {
  if (count == 0) return 0;
  u32 logn = 0;
  while ((1u << logn) < n) ++logn;
  ProfScope ps("k_fft_encode", s);
  if (n <= 8192) {
    const size_t sm = static_cast<size_t>(n) * sizeof(double2) * 3 / 2;  // array + n/2 roots
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_fft_encode<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           8192 * sizeof(double2) * 3 / 2);
      attr = true;
    }
    k_fft_encode<true><<<count, 1024, sm, s>>>(slots, n_slots, n, logn, level, scale, roots, twist, scratch, mags,
                                             max_mant, max_exp);
  } else if (n == 16384 && fft_cluster_on()) {
    const size_t sm = static_cast<size_t>(n / 2) * sizeof(double2);  // half the array per CTA
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_fft_encode2, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
      attr = true;
    }
    k_fft_encode2<<<count * 2, 1024, sm, s>>>(slots, n_slots, n, logn, level, scale, roots, twist, mags, max_mant,
                                              max_exp);
  } else {
    k_fft_encode<false><<<count, 512, 0, s>>>(slots, n_slots, n, logn, level, scale, roots, twist, scratch, mags,
                                              max_mant, max_exp);
  }
  return 1;
}

int launch_mags_to_residues(const ulonglong2* mags, u64 count, u32 n, u32 level, u32* out, const Basis& B,
                            cudaStream_t s) {
  const u64 total = count * n;
  if (total == 0) return 0;
  ProfScope ps("k_mags_to_residues", s);
  k_mags_to_residues<<<(total + 255) / 256, 256, 0, s>>>(mags, total, n, level, out, B);
  return 1;
}

double bench_int_peak(int device, int kind) {
  cudaSetDevice(device);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  u64* sink = nullptr;
  cudaMalloc(&sink, 8);
  const u32 iters = 2048;
  const int blocks = sms * 8, threads = 256;
  auto launch = [&](u32 it) {
    if (kind == 0) k_imad_probe<0><<<blocks, threads>>>(sink, it, 5);
    else if (kind == 1) k_imad_probe<1><<<blocks, threads>>>(sink, it, 5);
    else if (kind == 2) k_imad_probe<2><<<blocks, threads>>>(sink, it, 5);
    else k_imad_probe<3><<<blocks, threads>>>(sink, it, 5);
  };
  launch(16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    launch(iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  const double ops = static_cast<double>(blocks) * threads * iters * 16 * 8;
  return ops / (best * 1e-3);
}

}  // namespace hg
