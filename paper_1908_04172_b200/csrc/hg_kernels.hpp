// SPDX-License-Identifier: Apache-2.0
//
// Host-callable launchers for the sm_100a kernels in hg_kernels.cu.  Every
// launcher enqueues on `stream` and returns the number of kernel launches it
// issued (for the launch accounting reported by bench.py).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "hg_device.cuh"

namespace hg {

struct RescaleArgs {
  const u32* in;
  u32* out;
  u64 rows;  // ciphertexts * polys
  u32 level;  // input level (output level - 1 ... target)
  u32 pinv[kMaxPrimes];     // q_{level-1}^-1 mod q_i
  u32 pinv_sh[kMaxPrimes];
  u32 pm[kMaxPrimes];       // multiple of q_i >= floor(q_{level-1}/2): correction + pm >= 0
  int lazy;                 // every pm_i + floor(q_{level-1}/2) < 4 q_i: feed c + pm_i unreduced
  // Wide I/O (in64 != nullptr): the `level` limbs are limbs [io_off, io_off + level) of u64
  // rows of io_level_in limbs (output: io_level_out limbs), read and written in place
  const u64* in64;
  u64* out64;
  u32 io_level_in, io_level_out, io_off;
};

struct MacDenseArgs {
  const u32* X;     // [K][x_polys][x_level][N]
  u32* Y;           // [M][polys][level][N]
  const u32* W;     // [level][K][Mpad] weight residues
  const u32* bias;  // [level][Mpad] residues added to poly 0, or nullptr
  u32 K, M, Mpad, N;
  u32 level, polys;
  u32 x_level;      // limbs per polynomial in X (>= level)
  u32 fold[kMaxPrimes];  // 1 if limb i needs accumulator folding (products >= 2^48)
};

struct MacConvArgs {
  const u32* X;     // [C*IH*IW][polys][x_level][N]
  u32* Y;           // [F*OH*OW][polys][level][N]
  const u32* W;     // [level][F][C*win*win]
  const u32* bias;  // [level][F] or nullptr
  u32 C, IH, IW, F, OH, OW, win, stride, pad_top, pad_left;
  u32 level, polys, x_level, N;
  u32 fold[kMaxPrimes];
  u32 fp64[kMaxPrimes];  // taps * (q-1)^2 < 2^53 and taps <= 32: part of the MACs as exact DFMAs
  const u32* tap_off;    // [OH*OW + 1]: position p's valid taps are taps[tap_off[p] .. tap_off[p+1])
  const uint2* taps;     // (input word offset, window tap (c*win + ky)*win + kx), ascending per position
};

#ifndef HG_KEY_SHOUP
#define HG_KEY_SHOUP 0
#endif
// Relinearisation key layout: (value, Shoup companion) pairs, or values only (half the
// key-switch L1 traffic; the products then use the one-IMAD.HI product Barrett).
constexpr bool kKeyShoup = HG_KEY_SHOUP != 0;

// Relinearisation key columns t < chain_len stored pre-multiplied by P^-1 mod q_t (done once at
// upload): the key-switch accumulators then already carry the mod-down's 1/P, one modular
// product per coefficient and limb less in k_relin_moddown.  The special-prime column is
// unchanged (its accumulators are the mod-down's rounding corrections).
#ifndef HG_KEY_PINV
#define HG_KEY_PINV 1
#endif
constexpr bool kKeyPinv = HG_KEY_PINV != 0;

struct RelinArgs {
  const u32* A;   // mode 0: size-3 ciphertexts; mode 1: left operand (size 2)
  const u32* Bm;  // mode 1: right operand (size 2); may equal A (square)
  int mode;       // 0 = relinearize(ct3), 1 = relinearize(tensor(A, B))
  u64 count;
  u32 level;
  u32 chain_len;
  u32* D;         // digits   [count][level][N]
  u32* ACC;       // key-switch accumulators [count][2][level][N] (times P^-1 when kKeyPinv)
  i32* CORR;      // special-prime corrections [count][2][N]
  const void* key;   // [chain][2][chain+1][N]: uint2 (value, shoup) if kKeyShoup, else u32 value
  u32* out;       // [count][2][level or level-1][N]
  int rescale;
  u32 pinvP[kMaxPrimes], pinvP_sh[kMaxPrimes];  // P^-1 mod q_i
  u32 pinvL[kMaxPrimes], pinvL_sh[kMaxPrimes];  // q_{level-1}^-1 mod q_i
  u32 pmP[kMaxPrimes];  // multiple of q_i >= floor(P/2): special-prime correction + pmP >= 0
};

enum class EwOp : int { AddCC = 0, MulScalar = 1, AddScalar = 2, AddVector = 3, Tensor = 4, Copy = 5, GatherMul = 6 };

struct EwArgs {
  EwOp op;
  const u32* a;
  const u32* b;      // AddCC / Tensor: second ciphertext; AddVector: plaintexts [.][level][N]
  const u32* res;    // MulScalar / AddScalar: residues [.][level]
  int per_element;   // plaintext / residue indexed by element / pt_div (else broadcast)
  u32 pt_div;
  u32* out;
  u64 count;
  u32 polys_a, polys_out, level, N;
  // GatherMul: out[e] = a[gidx[e]] * res[gw[e]][limb] (zero where gidx[e] == ~0u)
  const u32* gidx;
  const u32* gw;
};

int launch_ntt(int logn, u32* data, u64 rows, u32 level, bool inverse, const Basis& B,
               cudaStream_t s);
int launch_rescale(int logn, const RescaleArgs& a, const Basis& B, cudaStream_t s);
// warps per CTA of the dense kernel for M outputs (BM = 4 * warps; Mpad must be a multiple of BM)
u32 mac_dense_warps(u32 M);
int launch_mac_dense(const MacDenseArgs& a, const Basis& B, cudaStream_t s);
int launch_mac_conv(const MacConvArgs& a, const Basis& B, cudaStream_t s);
int launch_relin(int logn, const RelinArgs& a, const Basis& B, cudaStream_t s);
int launch_elementwise(const EwArgs& a, const Basis& B, cudaStream_t s);

// u64 host words -> u32 device residues with the < q check; bad != 0 on violation.
int launch_narrow(const u64* in, u32* out, u64 words, u32 level, u32 N, const Basis& B,
                  int* d_bad, cudaStream_t s);
int launch_widen(const u32* in, u64* out, u64 words, cudaStream_t s);

// encode_scalar for `count` values.  out[limb * limb_stride + dst(v)] with
// dst(v) = (v / row_len) * row_stride + v % row_len.
int launch_encode_scalars_f32(const float* vals, u64 count, u32 row_len, u32 row_stride,
                              u64 limb_stride, u32 level, double scale, u32* out, const Basis& B,
                              cudaStream_t s);
int launch_encode_scalars_f64(const double* vals, u64 count, u32 row_len, u32 row_stride,
                              u64 limb_stride, u32 level, double scale, u32* out, const Basis& B,
                              cudaStream_t s);

// encode_vector front half: conj-extend, radix-2 DIT FFT in the reference's
// operation order, untwist, x87 scale/round -> signed 128-bit magnitudes
// (lo, hi | sign << 63) per coefficient.  max_mant/max_exp[pt] = the largest
// |scaled| as an exact long double (mantissa, exponent).
bool fft_cluster_on();  // 2-CTA cluster FFTs at n = 2^14 (HG_FFT_CLUSTER)
int launch_fft_encode(const double* slots, u32 n_slots, u64 count, u32 n, u32 level, double scale,
                      const double2* roots, const double2* twist, double2* scratch, ulonglong2* mags,
                      unsigned long long* max_mant, int* max_exp, cudaStream_t s);
int launch_mags_to_residues(const ulonglong2* mags, u64 count, u32 n, u32 level, u32* out, const Basis& B,
                            cudaStream_t s);

// Register-only integer pipe probe; kind 0 IMAD, 1 IMAD.WIDE, 2 IMAD.HI.  Lane-ops per second.
double bench_int_peak(int device, int kind);

// Brackets one kernel launch with CUDA events on its stream when profiling is on.
// Wraps exactly one kernel launch: counts it (launches_total) and, while the profiler is
// on, brackets it with CUDA events on its stream.
u64 launches_total();
struct ProfScope {
  const char* name;
  cudaStream_t s;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  ProfScope(const char* n, cudaStream_t st);
  ~ProfScope();
};

void prof_enable(bool on);
std::string prof_report();  // JSON: kernel -> {ms, launches}; clears the log

}  // namespace hg
