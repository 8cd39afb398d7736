// kv_append.cu -- direction-aware KV-cache write.
//
// in a shared block "KV cache of the RT request occupies memory
// slots from the left to the right ... that of the BE request in the opposite
// direction".  New token t of request r goes to block-table entry e = t / bs;
// slot t % bs for a forward (RT) entry, bs-1 - t % bs for a reversed (BE) one
// (direction table, readings Q3/Q4).  The copy is bit-exact.
//
// One CTA per request; each (token, head, K|V) row of head_dim bf16 is moved
// by head_dim/8 threads with one 16-byte load and one 16-byte store each, so a
// warp touches whole 128-byte lines on both sides.  The step is launch-latency
// bound (a decode step moves 4*B*H*d bytes); bkv_decode_step (f2) fuses the
// decode-step append into the attention kernel instead.
#include "bkv_internal.h"

namespace bkv {

// Fused lazy checkpoint ("only the KV tensors of a
// specific request that are about to be overwritten by its peer need to be
// checkpointed"): before new token i's row replaces a live peer row, the SAME
// thread copies the old 16 bytes out to checkpoint row evict[i] (device memory
// or the device alias of mapped pinned host memory), so program order alone
// orders the read before the overwrite.
template <int D>
__device__ __forceinline__ void evict_row(const AppendParams &p, int i, int h, int which, int sub,
                                          const uint16_t *slot_row) {
  const int er = __ldg(p.evict + i);
  if (er < 0) return;
  const uint4 old = *reinterpret_cast<const uint4 *>(slot_row);
  uint16_t *ck = which ? p.ck_v : p.ck_k;
  *reinterpret_cast<uint4 *>(ck + (static_cast<int64_t>(er) * p.H + h) * D + sub * 8) = old;
}

template <int D>
__global__ void __launch_bounds__(256) kv_append_kernel(AppendParams p) {
  constexpr int TPR = D / 8;  // threads per row, 16 B each
  // let a PDL-launched decode kernel start its seq_lens-only prologue now
  asm volatile("griddepcontrol.launch_dependents;");
  const int r = blockIdx.x;
  const int32_t first = p.cu_new[r];
  const int n = p.cu_new[r + 1] - first;
  if (n <= 0) return;
  const int before = p.before[r];
  const int sub = threadIdx.x % TPR;
  const int rows = n * p.H * 2;
  const int64_t bt_row = static_cast<int64_t>(r) * p.bt_stride;
  const int64_t dir_row = static_cast<int64_t>(r) * p.dir_rs;
  for (int row = threadIdx.x / TPR; row < rows; row += blockDim.x / TPR) {
    const int j = row / (2 * p.H);
    const int rem = row - j * 2 * p.H;
    const int which = rem / p.H;  // 0 = K, 1 = V
    const int h = rem - which * p.H;
    const int t = before + j;
    const int e = t / p.bs;
    const int within = t - e * p.bs;
    const int32_t blk = __ldg(p.bt + bt_row + e);
    const uint8_t dir = __ldg(p.dirs + dir_row + static_cast<int64_t>(e) * p.dir_cs);
    const int slot = dir ? (p.bs - 1 - within) : within;
    const int64_t src = (static_cast<int64_t>(first + j) * p.H + h) * D + sub * 8;
    const int64_t dst = static_cast<int64_t>(blk) * p.sb + static_cast<int64_t>(h) * p.sh +
                        static_cast<int64_t>(slot) * p.ss + sub * 8;
    const uint16_t *s = which ? p.v_new : p.k_new;
    uint16_t *d = which ? p.v : p.k;
    const uint4 val = __ldg(reinterpret_cast<const uint4 *>(s + src));
    if (p.evict) evict_row<D>(p, first + j, h, which, sub, d + dst);
    *reinterpret_cast<uint4 *>(d + dst) = val;
    if (p.slot_mapping && which == 0 && h == 0 && sub == 0)
      p.slot_mapping[first + j] = static_cast<int64_t>(blk) * p.bs + slot;
  }
}

// General map: entry e of request r holds n_e = fills[e]
// tokens, numbered in entry order, the j-th at slot j (forward) or bs-1-j
// (reversed).  The CTA builds the exclusive prefix F_e of
// the request's fills in shared memory (a block scan, 256 entries per pass);
// new token t then lives in the entry with F_e <= t < F_{e+1} (binary search),
// at j = t - F_e.  Copies as above: bit-exact, nothing else written.
template <int D>
__global__ void __launch_bounds__(256) kv_append_general_kernel(AppendParams p) {
  constexpr int TPR = D / 8;
  extern __shared__ int F[];   // [E + 1] exclusive prefix of the fills
  __shared__ int wsum[8];
  asm volatile("griddepcontrol.launch_dependents;");
  const int r = blockIdx.x;
  const int32_t first = p.cu_new[r];
  const int n = p.cu_new[r + 1] - first;
  if (n <= 0) return;
  const int E = p.nent[r];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint8_t *fr = p.fills + static_cast<int64_t>(r) * p.fill_rs;
  int carry = 0;
  for (int base = 0; base < E; base += 256) {
    const int e = base + static_cast<int>(threadIdx.x);
    const int v = e < E ? static_cast<int>(__ldg(fr + e)) : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    int before_w = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      before_w += w < warp ? wsum[w] : 0;
      tot += wsum[w];
    }
    if (e < E) F[e] = carry + before_w + x - v;
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) F[E] = carry;
  __syncthreads();
  const int before = p.before[r];
  const int sub = threadIdx.x % TPR;
  const int rows = n * p.H * 2;
  const int64_t bt_row = static_cast<int64_t>(r) * p.bt_stride;
  const int64_t dir_row = static_cast<int64_t>(r) * p.dir_rs;
  for (int row = threadIdx.x / TPR; row < rows; row += blockDim.x / TPR) {
    const int j = row / (2 * p.H);
    const int rem = row - j * 2 * p.H;
    const int which = rem / p.H;
    const int h = rem - which * p.H;
    const int t = before + j;
    int lo = 0, hi = E - 1;   // largest e in [0, E) with F[e] <= t
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (F[mid] <= t)
        lo = mid;
      else
        hi = mid - 1;
    }
    const int e = lo;
    const int within = t - F[e];
    const int32_t blk = __ldg(p.bt + bt_row + e);
    const uint8_t dir = __ldg(p.dirs + dir_row + static_cast<int64_t>(e) * p.dir_cs);
    const int slot = dir ? (p.bs - 1 - within) : within;
    const int64_t src = (static_cast<int64_t>(first + j) * p.H + h) * D + sub * 8;
    const int64_t dst = static_cast<int64_t>(blk) * p.sb + static_cast<int64_t>(h) * p.sh +
                        static_cast<int64_t>(slot) * p.ss + sub * 8;
    const uint16_t *s = which ? p.v_new : p.k_new;
    uint16_t *d = which ? p.v : p.k;
    const uint4 val = __ldg(reinterpret_cast<const uint4 *>(s + src));
    if (p.evict) evict_row<D>(p, first + j, h, which, sub, d + dst);
    *reinterpret_cast<uint4 *>(d + dst) = val;
    if (p.slot_mapping && which == 0 && h == 0 && sub == 0)
      p.slot_mapping[first + j] = static_cast<int64_t>(blk) * p.bs + slot;
  }
}

template <int D>
static cudaError_t launch_general(const AppendParams &p, cudaStream_t s) {
  const int smem = 4 * (p.max_entries + 1);
  if (smem > 48 * 1024) {
    cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void *>(kv_append_general_kernel<D>), smem);
    if (e != cudaSuccess) return e;
  }
  kv_append_general_kernel<D><<<p.B, 256, smem, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_kv_append(const AppendParams &p, int head_dim, cudaStream_t s) {
  if (p.B <= 0) return cudaSuccess;
  if (p.fills) return head_dim == 128 ? launch_general<128>(p, s) : launch_general<64>(p, s);
  dim3 grid(p.B), block(256);
  if (head_dim == 128)
    kv_append_kernel<128><<<grid, block, 0, s>>>(p);
  else
    kv_append_kernel<64><<<grid, block, 0, s>>>(p);
  return cudaGetLastError();
}

// Lazy checkpoint / restore: move the K and
// V rows of n arbitrary physical slots between the pool and a contiguous
// [n][H][d] buffer.  Grid-stride over (slot, head, K|V) rows, D/8 threads per
// row, one 16-byte load + store each.
template <int D>
__global__ void __launch_bounds__(256) slot_copy_kernel(SlotCopyParams p) {
  constexpr int TPR = D / 8;
  const int sub = threadIdx.x % TPR;
  const long long rows = static_cast<long long>(p.n) * p.H * 2;
  const long long stride = static_cast<long long>(gridDim.x) * (blockDim.x / TPR);
  for (long long row = blockIdx.x * (blockDim.x / TPR) + threadIdx.x / TPR; row < rows; row += stride) {
    const int i = static_cast<int>(row / (2 * p.H));
    const int rem = static_cast<int>(row - static_cast<long long>(i) * 2 * p.H);
    const int which = rem / p.H, h = rem - which * p.H;
    const int64_t sid = __ldg(p.slots + i);
    const int64_t blk = sid / p.bs, slot = sid - blk * p.bs;
    uint16_t *pool = which ? p.v : p.k;
    uint16_t *buf = which ? p.buf_v : p.buf_k;
    uint4 *pp = reinterpret_cast<uint4 *>(pool + blk * p.sb + h * p.sh + slot * p.ss + sub * 8);
    uint4 *bp = reinterpret_cast<uint4 *>(buf + (static_cast<int64_t>(i) * p.H + h) * D + sub * 8);
    if (p.restore)
      *pp = *bp;
    else
      *bp = *pp;
  }
}

cudaError_t launch_slot_copy(const SlotCopyParams &p, int head_dim, cudaStream_t s) {
  if (p.n <= 0) return cudaSuccess;
  const long long rows = static_cast<long long>(p.n) * p.H * 2;
  const int rows_per_cta = 256 / (head_dim / 8);
  const long long want = (rows + rows_per_cta - 1) / rows_per_cta;
  const int grid = static_cast<int>(want < 148 * 8 ? want : 148 * 8);
  if (head_dim == 128)
    slot_copy_kernel<128><<<grid, 256, 0, s>>>(p);
  else
    slot_copy_kernel<64><<<grid, 256, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace bkv
