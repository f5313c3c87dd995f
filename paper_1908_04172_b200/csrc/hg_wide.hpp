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
  // dropped prime >= 2^32: its centred corrections (|c| <= p/2) do not fit the i32 row in
  // shared memory; they go through this global scratch instead ([rows][N] i64)
  i64* corr64;
};

// Relinearization with u64 residues (henet/ckks.hpp:442-499) for any basis of primes
// < 2^62: the reference's algorithm in the NTT domain, three kernels
//   k_relin_digits_w  (ct, j):      digit j = INTT_j(c2_j)                 -> D
//   k_relin_keysw_w   (ct, t<=L):   acc_t = sum_j NTT_t(digit_j mod q_t) * key[j][.][t]
//                                   (t == L: the special prime P, whose accumulators are
//                                   INTT'd into the centred corrections c)  -> ACC, CORR
//   k_relin_moddown_w (ct, poly, i): out_i = c_poly,i + (acc_i - NTT_i(c mod q_i)) * P^-1
struct RelinArgsW {
  const u64* A;     // size-3 ciphertexts [count][3][level][N]
  u64* out;         // [count][2][level][N]
  u64* D;           // [count][level][N], coefficient domain
  u64* ACC;         // [count][2][level + 1][N]
  i64* CORR;        // [count][2][N]
  const u64* key;   // [chain][2][chain + 1][N]
  u64 count;
  u32 level, chain_len;
  u64 pinvP[kMaxPrimes], pinvP_sh[kMaxPrimes];  // P^-1 mod q_i and its 64-bit Shoup companion
};

struct MacDenseArgsW {
  const u64* X;
  u64* Y;
  const u64* W;     // [level][K][Mpad]
  const u64* bias;  // [level][Mpad] or nullptr
  u32 K, M, Mpad, N, level, polys, x_level;
  u32 limb_lo, limb_cnt;  // limbs computed: [limb_lo, limb_lo + limb_cnt); limb_cnt 0 = all
  uint8_t fold[kMaxPrimes];  // 1: K (q-1)^2 may overflow 128 bits -> reduce every 16 taps
};

struct MacConvArgsW {
  const u64* X;
  u64* Y;
  const u64* W;     // [level][F][C*win*win]
  const u64* bias;  // [level][F]
  u32 C, IH, IW, F, OH, OW, win, stride, pad_top, pad_left;
  u32 level, polys, x_level, N;
  uint8_t fold[kMaxPrimes];  // 1: taps (q-1)^2 may overflow 128 bits -> reduce every 8 taps
  // groups > 1: independent convolutions in one launch (a depthwise layer: one 1 -> 1
  // convolution per channel); group g reads X + g * gx, W + g * gw, bias + g * gb and writes
  // Y + g * gy (words)
  u32 groups;
  u64 gx, gy, gw, gb;
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
// first limb of the suffix of limbs below 2^30 (== level when there is none or no u32 basis)
u32 wide_narrow_lo(const BasisW& B, u32 level);
// decrypt's combine + INTT: limbs [0, lo) INTT'd in place in m (combined beforehand), limbs
// [lo, level) combined from ct / sk and INTT'd in one kernel; -2 when there is no such suffix
// encrypt's error NTT + combine: limbs [0, lo) NTT'd in place in err (combined afterwards),
// limbs [lo, level) transformed and combined into c0 in one kernel; -2 without such a suffix
int launch_enc_ntt_w(int logn, u64* ct, u64* err, const u64* pt, const u64* sk, u64 count, u32 level,
                     const BasisW& B, cudaStream_t s);
// encode's signed magnitudes -> NTT-domain residues: limbs [lo, level) reduced and transformed in
// one kernel, the wide limbs by k_mags_to_residues_w + the u64 NTT; -2 without such a suffix
int launch_pt_residues_ntt_w(int logn, const ulonglong2* mags, u64 count, u32 level, u64* out, const BasisW& B,
                             cudaStream_t s);
int launch_dec_intt_w(int logn, const u64* ct, const u64* sk, u64* m, u64 count, u32 polys, u32 level,
                      const BasisW& B, cudaStream_t s);
int launch_rescale_w(int logn, const RescaleArgsW& a, const BasisW& B, cudaStream_t s);
int launch_relin_w(int logn, const RelinArgsW& a, const BasisW& B, cudaStream_t s);
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
