// SPDX-License-Identifier: Apache-2.0
//
// Tensor-core (tcgen05.mma.kind::i8) dense modular contraction, hg_tc.cu.
#pragma once

#include <cuda_runtime.h>

#include "hg_kernels.hpp"

namespace hg {

struct MacDenseTcArgs {
  const u32* X;          // [K][x_polys][x_level][N]
  u32* Y;                // [M][polys][level][N]
  const uint8_t* Wp;     // packed weight byte planes (launch_pack_weights_tc)
  const u32* bias;       // [level][Mpad] or nullptr
  u32 K, M, Mpad, N, level, polys, x_level;
  u32 Mtiles, Ksteps;    // filled by the launcher
  // Wide I/O (X64 != nullptr): limbs [limb_off, limb_off + level) of u64 tensors are read and
  // written in place -- X64 [K][x_polys][x_level][N], Y64 [M][polys][y_level][N] -- instead
  // of X / Y; the Basis passed covers those limbs (index 0 = limb_off)
  const u64* X64;
  u64* Y64;
  u32 limb_off, y_level;
  u32 planes[kMaxPrimes];  // byte planes per limb: 3 if q < 2^24 else 4
  u32 cs[kMaxPrimes][8];   // 2^(8s) mod q per limb, s < 7, and 0 (filled by the launcher)
  // Batched contraction (a 1x1, stride-1 convolution: one Dot per output position): npos
  // positions; input k of position p is element k * x_kstride + p * x_pstride of X, output m
  // is element m * y_mstride + p * y_pstride of Y.  Zeros mean a plain Dot (1, 1, 0, 0).
  u32 npos;
  u64 x_kstride, x_pstride, y_mstride, y_pstride;
  u32 ppc;  // positions per CTA (filled by the launcher)
};

// One limb with a prime in [2^30, 2^40) (BASELINE c4/c5b limb 0), u64 residues: 5 byte
// planes, N tile 32 so the 9 diagonal accumulators fit in tensor memory.
struct MacDenseTcWArgs {
  const u64* X;          // [K][x_polys][x_level][N]
  u64* Y;                // [M][polys][level][N]
  const uint8_t* Wp;     // launch_pack_weights_tc_w
  const u64* bias;       // [Mpad] of this limb or nullptr
  u32 K, M, Mpad, N, level, polys, x_level, limb;
  u32 Mtiles, Ksteps;    // filled by the launcher
  u64 cs[10];            // 2^(8s) mod q, s < 9, and 0
  u32 npos;              // batched positions, as in MacDenseTcArgs
  u64 x_kstride, x_pstride, y_mstride, y_pstride;
  u32 ppc;               // positions per CTA (filled by the launcher)
};

u64 tc_packed_weight_bytes(u32 K, u32 M, u32 level);
u64 tc_packed_weight_bytes_w(u32 K, u32 M);
int launch_pack_weights_tc_w(const u64* W, uint8_t* Wp, u32 K, u32 M, u32 Mpad, cudaStream_t s);
// P: the limb's wide constants (hg_wide.cuh DevPrimeW, passed opaquely)
int launch_mac_dense_tc_w(MacDenseTcWArgs a, const void* P, cudaStream_t s);
int launch_pack_weights_tc(const u32* W, uint8_t* Wp, u32 K, u32 M, u32 Mpad, u32 level, cudaStream_t s);
int launch_mac_dense_tc(MacDenseTcArgs a, const Basis& B, cudaStream_t s);
double bench_tc_i8_peak(int device);  // measured kind::i8 MMA rate (MAC/s), roofline denominator

}  // namespace hg
