// SPDX-License-Identifier: Apache-2.0
//
// GPU encrypt / decrypt (hg_client.cu): the client side of henet/graph.hpp:68-103.
#pragma once

#include <cuda_runtime.h>

#include "hg_kernels.hpp"

namespace hg {

constexpr int kCrtWords = 8;   // Q < 2^512 (P14's 338-bit Q included)
constexpr int kCrtLimbs = 16;  // the GPU decoder's level limit (Q within kCrtWords words)

// Residue pointers are u32 words, or u64 words in wide contexts (the launchers' `wide`).
struct EncArgs {
  void* ct;         // [count][2][level][N]: c1 = a written by the sampler, c0 by combine
  void* err;        // [count][level][N]: error lifted into every limb (then NTT'd in place)
  const void* pt;   // [count][level][N]: encoded plaintexts (NTT domain)
  const void* sk;   // [full][N]: secret key s (NTT domain)
  int* flags;       // [count]: 1 if the counter-mode draw hit a rejection / u1 == 0
  u64 seed;         // encrypt_tensor seed; ciphertext e uses derive_seed(seed, e), stream 1
  u64 thr[kMaxPrimes];  // next_below rejection thresholds (2^64 mod q)
  u32 count, level, N;
  u32 e0;           // index of ciphertext 0 in the seed sequence (chunked refreshes)
  u32 limb_cnt;     // k_enc_combine: limbs [0, limb_cnt) only (0: all)
};

// Garner recomposition constants (k_dec_crt); passed by value next to the Basis, so only
// what the kernel reads is here.
struct CrtTables {
  u64 big_q[kCrtWords + 1];                 // Q = prod q_i
  u64 q_half[kCrtWords + 1];                // floor(Q / 2)
  u64 ginv[kCrtLimbs][kCrtLimbs];           // Garner: q_j^-1 mod q_i (j < i)
  u64 q[kCrtLimbs];                         // the level's primes
  // K-limb fast path (k_dec_crt): the centred CRT of (r_0 .. r_{K-1}) is the answer iff it
  // matches every other residue -- checked exactly.  fastk = 0 disables it.
  u32 fastk;
  u64 q01_lo, q01_hi;                       // q_0 .. q_{K-1}
  u64 q01_mod[kCrtLimbs];                   // q_0 .. q_{K-1} mod q_i
  u64 t64[kCrtLimbs];                       // 2^64 mod q_i (u32 contexts)
};

struct DecArgs {
  const void* ct;   // [count][polys][level][N]
  const void* sk;   // [full][N]
  void* m;          // [count][level][N]: decrypted plaintext residues
  double* coeffs;   // [count][N] (nullptr: residues only)
  u64 inv_mant;     // 1.0L / scale as an x87 long double: inv_mant * 2^inv_exp (host-computed)
  int inv_exp;
  CrtTables crt;
  u32 count, polys, level, N, words;
  u32 limb_cnt;     // k_dec_combine: limbs [0, limb_cnt) only (0: all)
};

int launch_batch_to_slots(const double* samples, u64 count, u64 e0, u32 cnt, u32 n_slots, int complex_pack,
                          double* slots, cudaStream_t s);
// B: the context's Basis, or its BasisW when `wide`
int launch_enc_sample(const EncArgs& a, const void* B, bool wide, cudaStream_t s);
// list == nullptr: walks the ciphertexts in [0, n_list) whose a.flags entry is set
int launch_enc_serial(const EncArgs& a, const u32* list, u32 n_list, const void* B, bool wide, cudaStream_t s);
int launch_enc_combine(const EncArgs& a, const void* B, bool wide, cudaStream_t s);
// decrypt (k_dec_combine) and, when a.coeffs is set, decode: INTT, CRT, forward embedding
// into slots [count][N/2][2]
int launch_dec(const DecArgs& a, int logn, const void* B, bool wide, const double2* roots, const double2* twist,
               double2* scratch, double* slots, cudaStream_t s);
// NonlinearityEngine::apply's per-slot function (henet/graph.hpp:714-731): slots
// [groups * window][N/2][2] -> [groups][N/2][2]; kind 1 = ReLU (window 1), 2 = max.
// clip > 0: ReLU is the clamp to [0, clip] (the ReLU6 refresh of BASELINE c4)
int launch_refresh_slots(const double* in, double* out, u32 groups, u32 window, u32 half, int kind, double clip,
                         cudaStream_t s);

}  // namespace hg
