// SPDX-License-Identifier: Apache-2.0
// Integer-pipe throughput probe for the NTT butterfly's instruction mix.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o int_pipe_probe int_pipe_probe.cu
// Each kernel runs 8 independent dependency chains per thread, 64 warps per SM;
// the printed rate is (chain steps) / s over the whole GPU.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

typedef uint32_t u32;
typedef uint64_t u64;

template <int KIND>
__global__ void probe(u32* sink, u32 iters, u32 seed) {
  u32 x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = (threadIdx.x ^ seed) * (2 * i + 3) + i;
  const u32 w = seed * 0x9e3779b1u, ws = seed * 0x85ebca6bu, q = 0x3fffc001u | seed;
  const double wq = 0.4375 + seed * 1e-9, cq = 4503599627370496.0 * (1.0 - wq);
  double dacc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) dacc[i] = 1.0 + i * seed;
  u64 a64[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a64[i] = x[i] * 3ull + i;
  for (u32 it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        u32 v = x[i];
        if (KIND == 0) {  // IMAD.HI chain: v = hi(v * ws)
          asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(v) : "r"(ws));
        } else if (KIND == 1) {  // IMAD chain: v = v * w
          asm volatile("mul.lo.u32 %0, %0, %1;" : "+r"(v) : "r"(w));
        } else if (KIND == 2) {  // IMAD.WIDE chain, high word: v = hi64(v * ws)
          u64 p;
          asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(v), "r"(ws));
          v = static_cast<u32>(p >> 32);
        } else if (KIND == 3) {  // Shoup lazy product, mul.hi form (3 multiplies)
          u32 h, lo;
          asm volatile("mul.hi.u32 %0, %1, %2;" : "=r"(h) : "r"(v), "r"(ws));
          asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(lo) : "r"(v), "r"(w));
          asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(v) : "r"(h), "r"(0u - q), "r"(lo));
        } else if (KIND == 4) {  // Shoup lazy product, mul.wide form
          u64 p;
          u32 lo;
          asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(v), "r"(ws));
          asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(lo) : "r"(v), "r"(w));
          asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(v) : "r"(static_cast<u32>(p >> 32)), "r"(0u - q), "r"(lo));
        } else if (KIND == 5) {  // IADD3 chain
          asm volatile("add.u32 %0, %0, %1;" : "+r"(v) : "r"(w));
        } else if (KIND == 6) {  // DFMA chain (rounded down), operand pair built from v
          double d = __hiloint2double(0x43300000, v);
          asm volatile("fma.rm.f64 %0, %0, %1, %2;" : "+d"(d) : "d"(wq), "d"(cq));
          v = __double2loint(d);
        } else if (KIND == 7) {  // Shoup with the quotient from one DFMA (pair + DFMA + 2 IMAD)
          double d = __hiloint2double(0x43300000, v);
          asm volatile("fma.rm.f64 %0, %0, %1, %2;" : "+d"(d) : "d"(wq), "d"(cq));
          const u32 h = __double2loint(d);
          u32 lo;
          asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(lo) : "r"(v), "r"(w));
          asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(v) : "r"(h), "r"(0u - q), "r"(lo));
        } else if (KIND == 9) {  // IMAD.WIDE accumulate chain (64-bit accumulator carried)
          u64 acc = (static_cast<u64>(x[(i + 1) & 7]) << 32) | v;
          asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc) : "r"(v), "r"(ws));
          v = static_cast<u32>(acc >> 32) ^ static_cast<u32>(acc);
        } else if (KIND == 10) {  // IMAD.WIDE with a register (opaque zero) addend, high word used
          u64 p;
          const u64 z = static_cast<u64>(seed >> 31);  // 0 at run time, opaque to the compiler
          asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(p) : "r"(v), "r"(ws), "l"(z));
          v = static_cast<u32>(p >> 32);
        } else if (KIND == 11) {  // IMAD.HI with a register addend
          asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(v) : "r"(ws), "r"(seed >> 31));
        } else if (KIND == 12) {  // Shoup with the quotient from mad.wide + register zero
          u64 p;
          u32 lo;
          const u64 z = static_cast<u64>(seed >> 31);
          asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(p) : "r"(v), "r"(ws), "l"(z));
          asm volatile("mul.lo.u32 %0, %1, %2;" : "=r"(lo) : "r"(v), "r"(w));
          asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(v) : "r"(static_cast<u32>(p >> 32)), "r"(0u - q), "r"(lo));
        } else if (KIND == 13) {  // IMAD.WIDE accumulate, multiplicand = another chain's low word
          asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(a64[i]) : "r"(static_cast<u32>(a64[(i + 3) & 7])), "r"(ws));
        } else if (KIND == 14) {  // pure DFMA chains (no integer work)
          asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(dacc[i]) : "d"(wq), "d"(cq));
        } else if (KIND == 15) {  // u32 -> f64 by I2F.F64.U32 + DADD into an accumulator
          dacc[i] += static_cast<double>(v);
          v += w;
        } else if (KIND == 16) {  // u32 -> f64 by the 2^52 pair trick (MOV + DADD)
          dacc[i] += __hiloint2double(0x43300000, v) - 4503599627370496.0;
          v += w;
        } else if (KIND == 8) {  // pure DFMA chain on doubles
          double d = __hiloint2double(v, v);
          asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(d) : "d"(wq), "d"(cq));
          v = __double2hiint(d) ^ __double2loint(d);
        }
        x[i] = v;
      }
    }
  }
  u32 s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s ^= x[i] ^ static_cast<u32>(a64[i] >> 17) ^ static_cast<u32>(dacc[i]);
  if (s == 0x12345u) sink[0] = s;
}

template <int KIND>
static double run(int sms) {
  u32* sink;
  cudaMalloc(&sink, 4);
  const int blocks = sms * 8, threads = 256;
  const u32 iters = 1024;
  probe<KIND><<<blocks, threads>>>(sink, 8, 7);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    probe<KIND><<<blocks, threads>>>(sink, iters, 7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  cudaFree(sink);
  const double steps = static_cast<double>(blocks) * threads * iters * 16 * 8;
  return steps / (best * 1e-3);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double per_clk = sms * (clk * 1e3);
  const char* names[] = {"IMAD.HI (mul.hi)", "IMAD (mul.lo)", "IMAD.WIDE hi (mul.wide)", "Shoup mul.hi form",
                         "Shoup mul.wide form", "IADD3", "pair+DFMA.RM", "Shoup DFMA quotient", "DFMA chain",
                         "IMAD.WIDE acc chain", "IMAD.WIDE reg-addend hi", "IMAD.HI reg-addend",
                         "Shoup mad.wide+reg0 form", "IMAD.WIDE accumulate (MAC)", "DFMA (pure)",
                         "I2F.F64 + DADD", "pair-MOV + 2 DADD"};
  double r[17] = {run<0>(sms),  run<1>(sms),  run<2>(sms),  run<3>(sms),  run<4>(sms),  run<5>(sms),
                  run<6>(sms),  run<7>(sms),  run<8>(sms),  run<9>(sms),  run<10>(sms), run<11>(sms),
                  run<12>(sms), run<13>(sms), run<14>(sms), run<15>(sms), run<16>(sms)};
  for (int k = 0; k < 17; ++k)
    printf("%-26s %8.2f T steps/s  %6.1f lanes/clk/SM\n", names[k], r[k] / 1e12, r[k] / per_clk);
  return 0;
}
