// SPDX-License-Identifier: Apache-2.0
//
// Launchers of the u64 ("wide") kernels in hg_wide.cu.  Argument structs mirror
// the u32 ones in hg_kernels.hpp with u64 residues.
#pragma once

#include <cuda_runtime.h>

#include "hg_kernels.hpp"
#include "hg_wide.cuh"
#include "hg_x87.cuh"

namespace hg {

struct RescaleArgsW {
  const u64* in;
  u64* out;
  u64 rows;
  u32 level;
  u32 limb_cnt;  // kept limbs computed: [0, limb_cnt); 0 = all (level - 1)
  u64 pinv[kMaxPrimes], pinv_sh[kMaxPrimes];
};

struct MacDenseArgsW {
  const u64* X;
  u64* Y;
  const u64* W;     // [level][K][Mpad]
  const u64* bias;  // [level][Mpad] or nullptr
  u32 K, M, Mpad, N, level, polys, x_level;
  u32 limb_lo, limb_cnt;  // limbs computed: [limb_lo, limb_lo + limb_cnt); limb_cnt 0 = all
};

struct MacConvArgsW {
  const u64* X;
  u64* Y;
  const u64* W;     // [level][F][C*win*win]
  const u64* bias;  // [level][F]
  u32 C, IH, IW, F, OH, OW, win, stride, pad_top, pad_left;
  u32 level, polys, x_level, N;
};

struct EwArgsW {
  EwOp op;
  const u64* a;
  const u64* b;
  const u64* res;
  int per_element;
  u32 pt_div;
  u64* out;
  u64 count;
  u32 polys_a, polys_out, level, N;
  const u32* gidx;  // GatherMul (EwArgs)
  const u32* gw;
};

int launch_ntt_w(int logn, u64* data, u64 rows, u32 level, bool inverse, const BasisW& B, cudaStream_t s);
int launch_rescale_w(int logn, const RescaleArgsW& a, const BasisW& B, cudaStream_t s);
u32 mac_dense_w_bm();  // Mpad must be a multiple of this
int launch_mac_dense_w(const MacDenseArgsW& a, const BasisW& B, cudaStream_t s);
// Limb range copies between u64 tensors [E][P][Lw][N] and u32 tensors [E][P][cnt][N]
// (limbs [lo, lo + cnt) of the wide layout; residues < 2^32, so the low word is exact).
int launch_limbs_to_u32(const u64* in, u32* out, u64 elems_polys, u32 Lw, u32 lo, u32 cnt, u32 N, cudaStream_t s);
int launch_limbs_to_u64(const u32* in, u64* out, u64 elems_polys, u32 Lw, u32 lo, u32 cnt, u32 N, cudaStream_t s);
int launch_mac_conv_w(const MacConvArgsW& a, const BasisW& B, cudaStream_t s);
int launch_elementwise_w(const EwArgsW& a, const BasisW& B, cudaStream_t s);
int launch_validate_w(const u64* w, u64 words, u32 level, u32 N, const BasisW& B, int* d_bad, cudaStream_t s);
int launch_encode_scalars_w_f32(const float* vals, u64 count, u32 row_len, u32 row_stride, u64 limb_stride, u32 level,
                                double scale, u64* out, const BasisW& B, cudaStream_t s);
int launch_encode_scalars_w_f64(const double* vals, u64 count, u32 row_len, u32 row_stride, u64 limb_stride,
                                u32 level, double scale, u64* out, const BasisW& B, cudaStream_t s);
int launch_mags_to_residues_w(const ulonglong2* mags, u64 count, u32 n, u32 level, u64* out, const BasisW& B,
                              cudaStream_t s);

}  // namespace hg
