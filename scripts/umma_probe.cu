// Dev probe (not product code): validates the tcgen05.mma / TMEM encodings the
// prefill kernel relies on, on one CTA, against a host reference.
//   S = Q.K^T   M=128, N=16, K=128: A = Q K-major SW128 (two 64-d halves),
//                                   B = K K-major SW128 ([half][16 slots][128B], as TMA lands it)
//   O = P.V     M=128, N=128, K=16: A = P K-major SW128 (128B rows, first 32B used),
//                                   B = V MN-major SW128 ([half][16 slots][128B])
//   O2 = P.V    the same product with A = P in TMEM (the "TS" form): row i = lane i,
//               bf16 pairs packed per 32-bit column (element k in column k/2, even
//               k in the low half), written by tcgen05.st from the row's thread
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_probe scripts/umma_probe.cu
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t swz(int row, int c) {   // 128B swizzle, 16B piece c of row
  return static_cast<uint32_t>(row * 128 + ((c ^ (row & 7)) << 4));
}
// SM100 shared-memory matrix descriptor (cute::UMMA::SmemDescriptor layout)
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;                 // version 1 (sm100)
  d |= (uint64_t)2 << 61;                 // SWIZZLE_128B
  return d;
}
// instruction descriptor: bf16 x bf16 -> f32, M, N, A/B major
__host__ __device__ constexpr uint32_t idesc(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D;\nbra W;\nD:\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void ld16(uint32_t taddr, float *v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__global__ void __launch_bounds__(128, 1) probe(const __nv_bfloat16 *Q, const __nv_bfloat16 *K,
                                                const __nv_bfloat16 *V, const __nv_bfloat16 *P,
                                                float *S_out, float *O_out, float *O2_out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *sQ = sm;                 // 2 halves x 128 rows x 128B = 32KB
  uint8_t *sK = sQ + 32768;         // 2 halves x 16 rows x 128B = 4KB
  uint8_t *sV = sK + 4096;          // 4KB
  uint8_t *sP = sV + 4096;          // 128 rows x 128B = 16KB
  uint64_t *bar = reinterpret_cast<uint64_t *>(sP + 16384);
  uint32_t *tslot = reinterpret_cast<uint32_t *>(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5;
  // fill smem with the swizzled layouts (16B pieces)
  for (int i = tid; i < 128 * 16; i += 128) {   // Q: row i/16, piece i%16 (d = 8*piece)
    const int row = i / 16, pc = i % 16;
    const uint4 v = reinterpret_cast<const uint4 *>(Q + row * 128)[pc];
    *reinterpret_cast<uint4 *>(sQ + (pc >> 3) * 16384 + swz(row, pc & 7)) = v;
  }
  for (int i = tid; i < 16 * 16; i += 128) {
    const int row = i / 16, pc = i % 16;
    *reinterpret_cast<uint4 *>(sK + (pc >> 3) * 2048 + swz(row, pc & 7)) = reinterpret_cast<const uint4 *>(K + row * 128)[pc];
    *reinterpret_cast<uint4 *>(sV + (pc >> 3) * 2048 + swz(row, pc & 7)) = reinterpret_cast<const uint4 *>(V + row * 128)[pc];
  }
  for (int i = tid; i < 128 * 8; i += 128) {    // P: 128 rows x 64 keys (first 16 real, rest 0)
    const int row = i / 8, pc = i % 8;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (pc < 2) v = reinterpret_cast<const uint4 *>(P + row * 16)[pc];
    *reinterpret_cast<uint4 *>(sP + swz(row, pc)) = v;
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tslot;
  const uint32_t tS = tmem, tO = tmem + 128, tP = tmem + 64, tO2 = tmem + 256;   // columns
  {   // P row tid -> TMEM lane tid, columns tP .. tP + 7 (bf16 pairs)
    uint32_t w[8];
    for (int c = 0; c < 8; ++c) {
      const __nv_bfloat162 pr = *reinterpret_cast<const __nv_bfloat162 *>(P + tid * 16 + 2 * c);
      w[c] = *reinterpret_cast<const uint32_t *>(&pr);
    }
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tP + lane_base),
                 "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    const uint32_t idS = idesc(128, 16, 0, 0), idO = idesc(128, 128, 0, 1);
    for (int k = 0; k < 8; ++k) {
      const uint32_t off = (k >> 2) * 0 + (k & 3) * 32;
      const uint64_t a = sdesc(smem_u32(sQ) + (k >> 2) * 16384 + off, 16, 1024);
      const uint64_t b = sdesc(smem_u32(sK) + (k >> 2) * 2048 + off, 16, 1024);
      mma(tS, a, b, idS, k > 0);
    }
    const uint64_t a = sdesc(smem_u32(sP), 16, 1024);
    const uint64_t b = sdesc(smem_u32(sV), 2048, 1024);
    mma(tO, a, b, idO, 0);
    mma_ts(tO2, tP, b, idO, 0);
    commit(smem_u32(bar));
  }
  mbar_wait(smem_u32(bar), 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int row = tid;   // warp w reads lanes 32w..32w+31
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  float v[16];
  ld16(tS + lane_base, v);
  for (int i = 0; i < 16; ++i) S_out[row * 16 + i] = v[i];
  for (int c = 0; c < 128; c += 16) {
    ld16(tO + lane_base + c, v);
    for (int i = 0; i < 16; ++i) O_out[row * 128 + c + i] = v[i];
    ld16(tO2 + lane_base + c, v);
    for (int i = 0; i < 16; ++i) O2_out[row * 128 + c + i] = v[i];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
  const int NQ = 128 * 128, NK = 16 * 128, NP = 128 * 16;
  __nv_bfloat16 *hQ = (__nv_bfloat16 *)malloc(NQ * 2), *hK = (__nv_bfloat16 *)malloc(NK * 2),
                *hV = (__nv_bfloat16 *)malloc(NK * 2), *hP = (__nv_bfloat16 *)malloc(NP * 2);
  srand(1);
  auto rnd = [] { return (float)(rand() % 2001 - 1000) / 500.f; };
  for (int i = 0; i < NQ; ++i) hQ[i] = __float2bfloat16(rnd());
  for (int i = 0; i < NK; ++i) hK[i] = __float2bfloat16(rnd()), hV[i] = __float2bfloat16(rnd());
  for (int i = 0; i < NP; ++i) hP[i] = __float2bfloat16(rnd());
  __nv_bfloat16 *dQ, *dK, *dV, *dP;
  float *dS, *dO, *dO2;
  cudaMalloc(&dQ, NQ * 2); cudaMalloc(&dK, NK * 2); cudaMalloc(&dV, NK * 2); cudaMalloc(&dP, NP * 2);
  cudaMalloc(&dS, 128 * 16 * 4); cudaMalloc(&dO, 128 * 128 * 4); cudaMalloc(&dO2, 128 * 128 * 4);
  cudaMemcpy(dQ, hQ, NQ * 2, cudaMemcpyHostToDevice); cudaMemcpy(dK, hK, NK * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dV, hV, NK * 2, cudaMemcpyHostToDevice); cudaMemcpy(dP, hP, NP * 2, cudaMemcpyHostToDevice);
  const int smem = 1024 + 32768 + 4096 + 4096 + 16384 + 64;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<<<1, 128, smem>>>(dQ, dK, dV, dP, dS, dO, dO2);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
  float *S = (float *)malloc(128 * 16 * 4), *O = (float *)malloc(128 * 128 * 4), *O2 = (float *)malloc(128 * 128 * 4);
  cudaMemcpy(O2, dO2, 128 * 128 * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(S, dS, 128 * 16 * 4, cudaMemcpyDeviceToHost); cudaMemcpy(O, dO, 128 * 128 * 4, cudaMemcpyDeviceToHost);
  double es = 0, eo = 0, eo2 = 0;
  for (int r = 0; r < 128; ++r)
    for (int c = 0; c < 16; ++c) {
      double ref = 0;
      for (int k = 0; k < 128; ++k) ref += (double)__bfloat162float(hQ[r * 128 + k]) * __bfloat162float(hK[c * 128 + k]);
      es = fmax(es, fabs(ref - S[r * 16 + c]));
    }
  for (int r = 0; r < 128; ++r)
    for (int c = 0; c < 128; ++c) {
      double ref = 0;
      for (int k = 0; k < 16; ++k) ref += (double)__bfloat162float(hP[r * 16 + k]) * __bfloat162float(hV[k * 128 + c]);
      eo = fmax(eo, fabs(ref - O[r * 128 + c]));
      eo2 = fmax(eo2, fabs(ref - O2[r * 128 + c]));
    }
  printf("S max err %.3e (S[0][0]=%f)  O max err %.3e (O[0][0]=%f)  O(TS, P in TMEM) max err %.3e (O2[0][0]=%f)\n",
         es, S[0], eo, O[0], eo2, O2[0]);
  printf("%s\n", (es < 1e-2 && eo < 1e-2 && eo2 < 1e-2) ? "UMMA PROBE OK" : "UMMA PROBE MISMATCH");
  return 0;
}
