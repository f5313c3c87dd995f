// SPDX-License-Identifier: Apache-2.0
//
// Pipe probe: can the FP64 pipe carry part of the NTT's modular products beside the IMAD
// (fmaheavy) pipe?  Register-only chains, 8 independent per thread, 148*8 CTAs of 256.
//   shoup:  x <- x*w - hi(x*w')*q                      (IMAD.HI + 2 IMAD)
//   fp64:   x <- fma(-rint(x*wq), q, x*w)  (exact for 24-bit q, |x| < 2^28)  (DMUL, DFMA+DADD, DFMA)
//   mixed:  K of the 8 chains Shoup, the rest FP64
//   cvt:    u32 -> f64 -> u32 round trip
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe scripts/fp64_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

typedef uint32_t u32;

template <int NSH>  // chains [0, NSH) Shoup, [NSH, 8) FP64
__global__ void k_probe(double* sink, u32 iters, u32 seed) {
  u32 a[8];
  double d[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i] = (threadIdx.x ^ seed) * (2 * i + 3) + i;
    d[i] = static_cast<double>((threadIdx.x * 7 + i) & 0xFFFFF);
  }
  const u32 wsh = seed * 0x9E3779B9u, w = seed | 1;
  const double q = 16760833.0, wd = static_cast<double>(seed & 0xFFFFFF), wq = wd / q;
  const double magic = 6755399441055744.0;  // 1.5 * 2^52
  for (u32 it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (i < NSH) {
          u32 x = a[i], h, lo;
          asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(h) : "r"(x), "r"(wsh));
          asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(lo) : "r"(x), "r"(w));
          asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(x) : "r"(h), "r"(0xc0004001u), "r"(lo));
          a[i] = x;
        } else {
          double x = d[i], t, k, y;
          asm volatile("mul.rn.f64 %0, %1, %2;" : "=d"(t) : "d"(x), "d"(wd));
          asm volatile("fma.rn.f64 %0, %1, %2, %3;" : "=d"(k) : "d"(x), "d"(wq), "d"(magic));
          asm volatile("sub.rn.f64 %0, %1, %2;" : "=d"(k) : "d"(k), "d"(magic));
          asm volatile("fma.rn.f64 %0, %1, %2, %3;" : "=d"(y) : "d"(k), "d"(-q), "d"(t));
          d[i] = y;
        }
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += (i < NSH) ? static_cast<double>(a[i]) : d[i];
  if (s == 1234.5) *sink = s;
}

__global__ void k_cvt(double* sink, u32 iters, u32 seed) {
  u32 a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = (threadIdx.x ^ seed) * (2 * i + 3) + i;
  for (u32 it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        double x;
        asm volatile("cvt.rn.f64.u32 %0, %1;" : "=d"(x) : "r"(a[i]));
        asm volatile("cvt.rzi.u32.f64 %0, %1;" : "=r"(a[i]) : "d"(x));
        a[i] ^= 1u;
      }
    }
  }
  u32 s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345u) *sink = s;
}

// 6 Shoup chains + 2 chains of one u32 -> f64 -> u32 round trip per step: do the
// conversions overlap the IMAD.HI pipe?
__global__ void k_shoup_cvt(double* sink, u32 iters, u32 seed) {
  u32 a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = (threadIdx.x ^ seed) * (2 * i + 3) + i;
  const u32 wsh = seed * 0x9E3779B9u, w = seed | 1;
  for (u32 it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (i < 6) {
          u32 x = a[i], h, lo;
          asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(h) : "r"(x), "r"(wsh));
          asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(lo) : "r"(x), "r"(w));
          asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(x) : "r"(h), "r"(0xc0004001u), "r"(lo));
          a[i] = x;
        } else {
          double x;
          asm volatile("cvt.rn.f64.u32 %0, %1;" : "=d"(x) : "r"(a[i]));
          asm volatile("cvt.rzi.u32.f64 %0, %1;" : "=r"(a[i]) : "d"(x));
          a[i] ^= 1u;
        }
      }
    }
  }
  u32 s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345u) *sink = s;
}

template <typename F>
double time_it(F launch) {
  launch(16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    launch(1024);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* sink;
  cudaMalloc(&sink, 8);
  const int blocks = sms * 8, threads = 256;
  const double chains = static_cast<double>(blocks) * threads * 1024 * 16;  // per chain slot
#define RUN(NSH)                                                                                      \
  {                                                                                                   \
    double ms = time_it([&](u32 it) { k_probe<NSH><<<blocks, threads>>>(sink, it, 5); });             \
    printf("shoup chains %d/8: %.3f ms  %.3f T modmul/s\n", NSH, ms, chains * 8 / (ms * 1e-3) / 1e12); \
  }
  RUN(8) RUN(7) RUN(6) RUN(5) RUN(4) RUN(3) RUN(0)
  double ms = time_it([&](u32 it) { k_cvt<<<blocks, threads>>>(sink, it, 5); });
  printf("cvt u32->f64->u32: %.3f ms  %.3f T round trips/s\n", ms, chains * 8 / (ms * 1e-3) / 1e12);
  ms = time_it([&](u32 it) { k_shoup_cvt<<<blocks, threads>>>(sink, it, 5); });
  printf("6 shoup + 2 cvt chains: %.3f ms  (6/8 shoup alone would be %.3f ms at the 8/8 rate)\n", ms,
         chains * 6 / 4.639e12 * 1e3);
  return 0;
}
