// mma_bench.cu — tcgen05.mma issue-rate microbenchmark (diagnostic, not product).
// Every CTA (one per SM) issues ITERS MMAs of shape M x N x 16 (bf16 -> fp32)
// back to back from one thread, committing to an mbarrier every 16 MMAs and
// waiting only for the last commit. Variants: A from TMEM ("ts") or SMEM
// ("ss"), N in {64, 128, 256}, cta_group::1. Prints TFLOP/s per variant.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_bench mma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

template <int N, bool TS, int NACC>
__global__ void __launch_bounds__(128, 1) k_mma(int iters, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((uint32_t*)base)[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const uint64_t bd = desc_sw128(smem_u32(base));
    const uint64_t ad = desc_sw128(smem_u32(base + 32768));
    for (int it = 0; it < iters; ++it) {
      const uint32_t d_tmem = tmem + 256 - (NACC > 1 && NACC < 9 ? 256 : 0) + (it % (NACC == 9 ? 1 : NACC)) * N;  // NACC>1: accs from col 0
      const uint32_t acc = it & 15 ? 1u : 0u;
      if (NACC == 9) {  // 4 MMAs in one asm block, uniform operands, no per-MMA loop code
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n}" ::"r"(tmem + 256),
            "l"(ad), "l"(bd), "r"(idesc), "r"(acc)
            : "memory");
        it += 3;
      } else if (TS) {
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d_tmem),
            "r"(tmem + (it & 3) * 8), "l"(bd + (it & 3) * 2), "r"(idesc), "r"(acc)
            : "memory");
      } else {
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
            "l"(ad + (it & 3) * 2), "l"(bd + (it & 3) * 2), "r"(idesc), "r"(acc)
            : "memory");
      }
      if ((it & 15) == 15 || (NACC == 9 && (it & 15) == 15))
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                     : "memory");
    }
  }
  __syncwarp();
  if (warp == 0) {
    // wait for the final commit phase: iters/16 commits -> parity of the last
    const uint32_t phase = ((iters / 16) - 1) & 1;
    asm volatile(
        "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}" ::"r"(
            smem_u32(&bar)),
        "r"(phase)
        : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
  if (threadIdx.x == 0 && sink) sink[blockIdx.x] = 0.f;
}

template <int N, bool TS, int NACC = 1>
void run(int sms) {
  const int iters = 16 * 4096;
  auto k = k_mma<N, TS, NACC>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024 + 1024);
  k<<<sms, 128, 64 * 1024 + 1024>>>(1024, nullptr);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<<<sms, 128, 64 * 1024 + 1024>>>(iters, nullptr);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double flops = 2.0 * 128 * N * 16 * (double)iters * sms;
  printf("M=128 N=%3d nacc=%d %s: %.3f ms  %.1f TFLOP/s  (%.1f cyc/MMA @1.965GHz)  err=%s\n", N, NACC, TS ? "A:tmem" : "A:smem", ms,
         flops / (ms * 1e-3) / 1e12, ms * 1e-3 * 1.965e9 / iters, cudaGetErrorString(cudaGetLastError()));
}

// cta_group::2: M=256 (128 rows per CTA), A and B from SMEM, leader issues.
template <int N, int NACC, bool I8 = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k_mma2(int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) ((uint32_t*)base)[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if (rank == 0 && threadIdx.x == 0) {
    // kind::i8: D s32 (2 << 4), A/B signed 8-bit (1 << 7, 1 << 10), K = 32 per MMA
    const uint32_t idesc = I8 ? ((2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24))
                              : ((1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24));
    const uint64_t bd = desc_sw128(smem_u32(base));
    const uint64_t ad = desc_sw128(smem_u32(base + 32768));
    for (int it = 0; it < iters; ++it) {
      const uint32_t d_tmem = tmem + (it % NACC) * N;
      const uint32_t acc = it & 15 ? 1u : 0u;
      if (I8)
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
          "l"(ad + (it & 3) * 2), "l"(bd + (it & 3) * 2), "r"(idesc), "r"(acc)
          : "memory");
      else
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
          "l"(ad + (it & 3) * 2), "l"(bd + (it & 3) * 2), "r"(idesc), "r"(acc)
          : "memory");
      if ((it & 15) == 15)
        asm volatile(
            "{\n.reg .b16 m;\nmov.b16 m, 3;\n"
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n}" ::"r"(
                smem_u32(&bar))
            : "memory");
    }
  }
  __syncwarp();
  if (warp == 0) {
    const uint32_t phase = ((iters / 16) - 1) & 1;
    asm volatile(
        "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W;\n}" ::"r"(
            smem_u32(&bar)),
        "r"(phase)
        : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int N, int NACC, bool I8 = false>
void run_pair(int sms) {
  const int iters = 16 * 4096;
  auto k = k_mma2<N, NACC, I8>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024 + 1024);
  k<<<sms, 128, 64 * 1024 + 1024>>>(1024);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<<<sms, 128, 64 * 1024 + 1024>>>(iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double flops = 2.0 * 256 * N * (I8 ? 32 : 16) * (double)iters * (sms / 2);
  printf("PAIR %s M=256 N=%3d nacc=%d: %.3f ms  %.1f T(FL)OP/s  (%.1f cyc/MMA)  err=%s\n", I8 ? "i8  " : "bf16", N, NACC, ms,
         flops / (ms * 1e-3) / 1e12, ms * 1e-3 * 1.965e9 / iters, cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  if (argc > 1) {  // "i8": int8 vs bf16 pair rates only
    for (int rep = 0; rep < 2; ++rep) {
      run_pair<128, 2>(sms);
      run_pair<128, 2, true>(sms);
      run_pair<256, 1, true>(sms);
      run_pair<256, 2, true>(sms);
      run_pair<64, 2, true>(sms);
    }
    return 0;
  }
  run<64, false, 9>(sms);
  run<128, false, 9>(sms);
  run<32, false, 9>(sms);
  run<64, true>(sms);
  run<64, false, 2>(sms);
  run<64, false, 4>(sms);
  run<128, false>(sms);
  run<128, false, 2>(sms);
  run<128, false, 4>(sms);
  run<256, false>(sms);
  run<256, false, 2>(sms);
  run_pair<64, 1>(sms);
  run_pair<64, 2>(sms);
  run_pair<128, 1>(sms);
  run_pair<128, 2>(sms);
  run_pair<256, 1>(sms);
  return 0;
}
