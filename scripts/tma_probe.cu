// tma_probe.cu -- dev microbenchmark: read bandwidth of per-warp TMA rings on
// B200 as a function of warps/SM, ring depth and box size, with random 4 KiB
// block order (the paged-KV access pattern).  Not part of the product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_probe tma_probe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>
#include <algorithm>
#include <random>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// mode 0: 1-D bulk copy of `box` bytes; mode 1: per-lane 16-B LDG into registers (sum)
__global__ void probe(const uint8_t *__restrict__ buf, const int *__restrict__ order, int nblk,
                      int blk_bytes, int S, int mode, int iters, unsigned long long *sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int W = blockDim.x / 32, warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  uint8_t *ring = smem + warp * S * blk_bytes;
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + W * S * blk_bytes) + warp * S;
  const int gw = blockIdx.x * W + warp, TW = gridDim.x * W;
  unsigned long long acc = 0;
  if (mode == 0 || mode == 2 || mode == 3) {
    if (lane == 0)
      for (int i = 0; i < S; ++i)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bars + i)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    // block ids for 32 future iterations live in lane registers (no global
    // load on the issue path), refilled warp-wide every 32 iterations
    int win_base = -1000000, win = 0;
    auto issue = [&](int k, int slot) {
      if (k - win_base >= 32) {
        win_base = k;
        win = order[(gw + (long long)(k + lane) * TW) % nblk];
      }
      const int b = __shfl_sync(0xffffffffu, win, k - win_base);
      if (lane == (mode == 2 ? slot % 32 : 0)) {
        const uint32_t bar = smem_u32(bars + slot);
        asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(blk_bytes) : "memory");
        if (mode == 3) {   // the same bytes as two half-size copies on one barrier
          const int hb = blk_bytes / 2;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(ring + slot * blk_bytes)),
                       "l"(buf + (size_t)b * blk_bytes), "r"(hb), "r"(bar) : "memory");
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(ring + slot * blk_bytes + hb)),
                       "l"(buf + (size_t)b * blk_bytes + hb), "r"(hb), "r"(bar) : "memory");
        } else {
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(ring + slot * blk_bytes)),
                       "l"(buf + (size_t)b * blk_bytes), "r"(blk_bytes), "r"(bar) : "memory");
        }
      }
    };
    for (int k = 0; k < S && k < iters; ++k) issue(k, k);
    for (int k = 0; k < iters; ++k) {
      const int slot = k % S;
      const uint32_t ph = (k / S) & 1;
      asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(smem_u32(bars + slot)), "r"(ph) : "memory");
      acc += ring[slot * blk_bytes + lane * 4];
      __syncwarp();
      if (k + S < iters) issue(k + S, slot);
    }
  } else {
    for (int k = 0; k < iters; ++k) {
      const int b = order[(gw + (long long)k * TW) % nblk];
      const uint4 *src = reinterpret_cast<const uint4 *>(buf + (size_t)b * blk_bytes);
      for (int i = lane; i < blk_bytes / 16; i += 32) {
        uint4 v;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(src + i));
        acc += v.x ^ v.w;
      }
    }
  }
  if (acc == 0x123456789ull) sink[0] = acc;
}

int main() {
  const size_t total = 4ull << 30;   // 4 GiB >> L2
  uint8_t *buf;
  cudaMalloc(&buf, total);
  cudaMemset(buf, 1, total);
  unsigned long long *sink;
  cudaMalloc(&sink, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  printf("mode blk_KB W S  GB/s\n");
  for (int mode : {3, 0})
    for (int blk : {8192, 16384}) {
      const int nblk = (int)(total / blk);
      std::vector<int> order(nblk);
      for (int i = 0; i < nblk; ++i) order[i] = i;
      std::shuffle(order.begin(), order.end(), std::mt19937(1));
      int *dorder;
      cudaMalloc(&dorder, nblk * 4);
      cudaMemcpy(dorder, order.data(), nblk * 4, cudaMemcpyHostToDevice);
      for (int W : {1, 4, 8})
        for (int S : {1, 2, 4}) {
          if (mode == 1 && S > 1) continue;
          const size_t smem = (size_t)W * S * blk + W * S * 8 + 64;
          if (mode != 1 && smem > 220 * 1024) continue;
          const long long per_warp = (long long)nblk / (sms * W);
          const int iters = (int)std::min<long long>(per_warp, 2000);
          cudaEvent_t a, b;
          cudaEventCreate(&a);
          cudaEventCreate(&b);
          probe<<<sms, W * 32, mode != 1 ? smem : 0>>>(buf, dorder, nblk, blk, S, mode, iters, sink);
          cudaEventRecord(a);
          probe<<<sms, W * 32, mode != 1 ? smem : 0>>>(buf, dorder, nblk, blk, S, mode, iters, sink);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          const double bytes = (double)sms * W * iters * blk;
          printf("%s %5d %2d %d  %7.0f   %s\n", mode == 1 ? "ldg " : (mode == 3 ? "bulk2" : "bulk"), blk / 1024, W, S, bytes / ms / 1e6,
                 cudaGetErrorString(cudaGetLastError()));
        }
      cudaFree(dorder);
    }
  return 0;
}
