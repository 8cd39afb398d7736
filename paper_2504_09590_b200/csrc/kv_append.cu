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
// bound (a decode step moves 4*B*H*d bytes); NEXT f2 fuses it into attention.
#include "bkv_internal.h"

namespace bkv {

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
    *reinterpret_cast<uint4 *>(d + dst) = val;
    if (p.slot_mapping && which == 0 && h == 0 && sub == 0)
      p.slot_mapping[first + j] = static_cast<int64_t>(blk) * p.bs + slot;
  }
}

cudaError_t launch_kv_append(const AppendParams &p, int head_dim, cudaStream_t s) {
  if (p.B <= 0) return cudaSuccess;
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
