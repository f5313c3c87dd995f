// SPDX-License-Identifier: Apache-2.0
// Raw tcgen05.mma.kind::i8 throughput with the operand layout of hg_tc.cu (K-major,
// SWIZZLE_NONE core matrices, LBO 128 B, SBO 256 B): one CTA per SM issues back-to-back
// M=128 x N x K=32 MMAs from static shared-memory operands (no producers, no epilogue).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_probe umma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

typedef uint32_t u32;
typedef uint64_t u64;

__device__ __forceinline__ u32 smem_addr(const void* p) { return static_cast<u32>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ u64 desc(u32 saddr) {
  return static_cast<u64>((saddr >> 4) & 0x3FFF) | (static_cast<u64>(128 >> 4) << 16) |
         (static_cast<u64>(256 >> 4) << 32) | (1ull << 46);
}

template <int NN>
__global__ void __launch_bounds__(128, 1) probe(u32 iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* A = sm;             // 128 x 32 B
  uint8_t* Bm = sm + 4096;     // NN x 32 B
  __shared__ u32 tmem;
  __shared__ __align__(8) unsigned long long bar;
  for (u32 i = threadIdx.x; i < (4096 + NN * 32) / 4; i += blockDim.x) reinterpret_cast<u32*>(sm)[i] = i * 2654435761u;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_addr(&tmem)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_addr(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::);
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
  if (threadIdx.x == 0) {
    const u32 idesc = (2u << 4) | ((NN >> 3) << 17) | ((128 >> 4) << 24);
    const u64 ad = desc(smem_addr(A)), bd = desc(smem_addr(Bm));
    const u64 t0 = clock64();
    for (u32 it = 0; it < iters; ++it) {
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc),
          "r"(it));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_addr(&bar)));
    asm volatile(
        "{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(
            smem_addr(&bar)));
    cycles[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
}

template <int NN>
static void run(int sms) {
  unsigned long long* d;
  cudaMalloc(&d, sms * 8);
  const size_t smem = 4096 + NN * 32;
  cudaFuncSetAttribute(probe<NN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const u32 iters = 20000;
  probe<NN><<<sms, 128, 200 * 1024>>>(100, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<NN><<<sms, 128, 200 * 1024>>>(iters, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long c;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  const double macs = static_cast<double>(sms) * iters * 128.0 * NN * 32.0;
  printf("N=%3d: %.1f cycles/MMA (SM 0), %.0f T int8 MAC/s over the GPU (%s)\n", NN, double(c) / iters,
         macs / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  (void)smem;
  cudaFree(d);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<256>(sms);
  run<192>(sms);
  run<128>(sms);
  run<64>(sms);
  return 0;
}
