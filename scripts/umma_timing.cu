// Dev probe (not product code): issue-to-completion time of tcgen05.mma batches on
// one CTA (one SM), to size the prefill kernel's pipeline.  Operands are garbage
// (timing only).  Build/run:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/umma_timing scripts/umma_timing.cu && /tmp/umma_timing
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__host__ __device__ constexpr uint32_t idesc(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t id) {
  asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n}\n" ::"r"(d), "l"(a), "l"(b), "r"(id) : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id) {
  asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;\n}\n" ::"r"(d), "r"(a), "l"(b), "r"(id) : "memory");
}
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(bar), "r"(parity) : "memory");
}

// 8 SS MMAs issued from ONE asm block under one elect (descriptors as operands)
__device__ __forceinline__ void mma8_ss(uint32_t d, const uint64_t (&a)[8], const uint64_t (&b)[8], uint32_t id) {
  asm volatile("{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
               "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %9, %17, 0;\n"
               "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %10, %17, 1;\n"
               "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %3, %11, %17, 1;\n"
               "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %4, %12, %17, 1;\n"
               "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %5, %13, %17, 1;\n"
               "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %6, %14, %17, 1;\n"
               "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %7, %15, %17, 1;\n"
               "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %8, %16, %17, 1;\n}\n" ::"r"(d),
               "l"(a[0]), "l"(a[1]), "l"(a[2]), "l"(a[3]), "l"(a[4]), "l"(a[5]), "l"(a[6]), "l"(a[7]),
               "l"(b[0]), "l"(b[1]), "l"(b[2]), "l"(b[3]), "l"(b[4]), "l"(b[5]), "l"(b[6]), "l"(b[7]), "r"(id)
               : "memory");
}

// mode 0: SS M128 N=n K16 (A K-major 128 rows, B K-major n rows); mode 1: TS (A from TMEM)
__global__ void probe(int mode, int n, int count, int reps, long long *out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const uint32_t base = (smem_u32(sm) + 1023) & ~1023u;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tslot;
  if (threadIdx.x < 32) {
    const uint32_t id = mode != 1 ? idesc(128, n, 0, 0) : idesc(128, n, 0, 1);
    long long tot = 0, first = 0;
    uint64_t da[8], db[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      da[k] = sdesc(base + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
      db[k] = sdesc(base + 65536 + (k >> 2) * 8192 + (k & 3) * 32, 16, 1024);
    }
    for (int r = 0; r < reps; ++r) {
      const long long t0 = clock64();
      if (mode == 2) {
        for (int i = 0; i < count; i += 8) mma8_ss(tm + (i & 8) * 32, da, db, id);
      } else if (mode == 3) {
        for (int i = 0; i < count; i += 8) {
#pragma unroll
          for (int k = 0; k < 8; ++k) mma_ss(tm + (i & 8) * 32, da[k], db[k], id);
        }
      } else
      for (int i = 0; i < count; ++i) {
        const uint64_t b = sdesc(base + 65536 + (i & 3) * 32, 16, 1024);
        if (mode == 0) mma_ss(tm + (i & 1) * 256, sdesc(base + (i & 3) * 32, 16, 1024), b, id);
        else mma_ts(tm + 256, tm + (i & 7) * 8, sdesc(base + 65536 + (i & 3) * 2048, 8192, 1024), id);
      }
      const long long t1 = clock64();
      commit(smem_u32(&bar));
      mbar_wait(smem_u32(&bar), r & 1);
      const long long t2 = clock64();
      if (r == 0) first = t2 - t0;
      else tot += t2 - t0;
      if (threadIdx.x == 0 && r == reps - 1) { out[0] = t1 - t0; out[1] = t2 - t0; }
    }
    if (threadIdx.x == 0) { out[2] = tot / (reps - 1); out[3] = first; }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
  long long *d, h[4];
  cudaMalloc(&d, 64);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int mode = 0; mode < 4; ++mode)
    for (int n : {64, 128, 256})
      for (int count : {8, 64}) {
        if (mode >= 2 && count < 8) continue;
        probe<<<1, 128, 200 * 1024>>>(mode, n, count, 20, d);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
        const double flop = 2.0 * 128 * n * 16 * count;
        printf("%s N=%3d count=%2d: issue %5lld cyc, issue->done %6lld cyc (first rep %6lld), %.0f FLOP/cyc  %s\n",
               mode == 0 ? "SS" : mode == 1 ? "TS" : mode == 2 ? "SS8asm" : "SSunroll", n, count, h[0], h[2], h[3], flop / h[2], e ? cudaGetErrorString(e) : "");
      }
  return 0;
}
