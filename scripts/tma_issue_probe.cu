// tma_issue_probe.cu -- dev microbenchmark: issue cost (SM cycles, issuing
// thread) of TMA tensor loads, 1-D bulk copies and mbarrier arrives on sm_100a.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_issue_probe tma_issue_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ CUtensorMap tm, const uint8_t *src, long long *out, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const int N = 16;
  if (threadIdx.x == 0) {
    const uint32_t b = su32(&bar);
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(N * 4096) : "memory");
    long long t0 = clock64();
    for (int i = 0; i < N; ++i) {
      const uint32_t dst = su32(sm + i * 4096);
      if (mode == 0) {
        asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4, %5, %6}], [%7], %8;"
                     ::"r"(dst), "l"(&tm), "r"(0), "r"(0), "r"(0), "r"(i), "r"(blockIdx.x), "r"(b), "l"(pol) : "memory");
      } else if (mode == 1) {
        asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                     ::"r"(dst), "l"(&tm), "r"(0), "r"(0), "r"(0), "r"(i), "r"(blockIdx.x), "r"(b) : "memory");
      } else {
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(dst), "l"(src + ((size_t)blockIdx.x * N + i) * 4096), "r"(4096), "r"(b) : "memory");
      }
    }
    long long t1 = clock64();
    asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(b) : "memory");
    long long t2 = clock64();
    out[blockIdx.x * 2] = t1 - t0;
    out[blockIdx.x * 2 + 1] = t2 - t0;
  }
}

int main() {
  const int nb = 148, N = 16;
  const size_t bytes = (size_t)nb * N * 4096 * 4;
  uint8_t *buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 0, bytes);
  long long *out;
  cudaMalloc(&out, nb * 16);
  void *fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fp;
  CUtensorMap tm;
  // (64, 16 slots, 2 halves, 16 heads, nb blocks) like the decode pool, bf16
  cuuint64_t dims[5] = {64, 16, 2, (cuuint64_t)N, (cuuint64_t)nb};
  cuuint64_t strides[4] = {256, 128, 4096, (cuuint64_t)N * 4096};
  cuuint32_t box[5] = {64, 16, 2, 1, 1}, es[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, N * 4096 + 1024);
  const char *names[3] = {"tensor5d+hint", "tensor5d", "bulk1d"};
  for (int mode = 0; mode < 3; ++mode)
    for (int rep = 0; rep < 3; ++rep) {
      k<<<nb, 32, N * 4096 + 1024>>>(tm, buf, out, mode);
      cudaDeviceSynchronize();
      long long h[nb * 2];
      cudaMemcpy(h, out, sizeof h, cudaMemcpyDeviceToHost);
      double is = 0, tot = 0;
      for (int i = 0; i < nb; ++i) { is += h[2 * i]; tot += h[2 * i + 1]; }
      printf("%-14s rep %d: issue %.0f cycles per copy, all-%d-landed %.0f cycles  (%s)\n", names[mode], rep, is / nb / N, N,
             tot / nb, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
