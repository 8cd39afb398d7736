// prefill_attention.cu -- mixed prefill + decode attention over BROS's
// bidirectional paged KV cache.
//
// BROS concatenates "the prefill requests followed by the decode requests",
// keeps a length table and dispatches each part to an attention kernel
// (the paper used xformers for the prefill part).  Here ONE
// kernel serves both parts straight from the shared paged blocks: request r
// has L = seq_lens[r] resident tokens (its new ones already appended, reading
// Q7) and its LAST n = cu_q[r+1] - cu_q[r] tokens are queries; query i is
// logical token p = L - n + i and attends causally to tokens t <= p
// (a decode request is n = 1).
//
// Design (B200, DESIGN.md §6 "prefill attention"):
//  * One CTA per (128-row query tile, kv head, request); rows are (token,
//    q-head-of-the-group) pairs, row = token*g + j, so a GQA group shares every
//    K/V tile it streams.  Tiles run longest-first (reversed causal order).
//  * A producer warp walks the request's block-table entries in logical order
//    (dense map: entry e holds tokens [e*bs, ...); general map (f3): prefix of
//    the fill counts) and streams each 16-slot chunk's K and V tiles with one
//    5-D TMA load each (128B swizzle, same tensor maps as decode) into a 4-stage
//    mbarrier ring (full: TMA bytes, empty: one arrive per consumer warp);
//    chunks whose first live token lies past the tile's last query position
//    are never loaded.  Each stage's chunk metadata (live slot range, token of
//    slot 0, direction) is handed to the consumers through a named barrier.
//  * 8 consumer warps, 16 rows each, FA2-style on bf16 mma.sync m16n8k16 with
//    fp32 accumulation: S = Q.K^T (Q fragments in registers, K via ldmatrix),
//    causal + direction mask by token index (slot s of a chunk holds token
//    base + s forward or base - s reversed), online softmax in the
//    log2 domain, P re-used from the S accumulators as the A operand, V via
//    ldmatrix.trans.  Dead slots (outside the entry's live range) are never
//    combined arithmetically: their scores are selected to -inf and their V
//    fragment halves are masked to zero before the MMA (reading Q10).
#include <math.h>
#include <stdlib.h>

#include "bkv_internal.h"
#include "bkv_ptx.cuh"

namespace bkv {

namespace {

constexpr int kStages = 4;
constexpr int kConsumerWarps = 8;
constexpr int kRowsPerTile = 16 * kConsumerWarps;
constexpr int kLast = 1 << 8;   // chunk-metadata flag: no more chunks

__device__ __forceinline__ uint32_t pswz(int row, int c) {
  return static_cast<uint32_t>(row * 128 + ((c ^ (row & 7)) << 4));
}

// The request's 16-slot chunks in logical entry order, skipping dead chunks
// and chunks whose first live token lies past the tile's last query (run by the
// producer warp).  Entries are read 32 at a time into a lane-distributed window
// (lane i: entry wb + i) and broadcast by shuffle, keeping global-load latency
// off the per-chunk path.
struct ChunkWalk {
  int e, c, F, E, wb;    // entry, chunk in entry, first token of entry, entries, window base
  int wblk, wdir, wfill; // this lane's window entry
  int blk, dir, fill;    // current entry (warp-uniform)
  bool have;
};

__device__ __forceinline__ void walk_window(const PrefillParams &p, int r, int L, ChunkWalk &w, int wb) {
  const int e = wb + static_cast<int>(threadIdx.x & 31);
  w.wb = wb;
  w.wblk = w.wdir = w.wfill = 0;
  if (e < w.E) {
    w.wblk = __ldg(p.bt + static_cast<int64_t>(r) * p.bt_stride + e);
    w.wdir = __ldg(p.dirs + static_cast<int64_t>(r) * p.dir_rs + static_cast<int64_t>(e) * p.dir_cs);
    w.wfill = p.fills ? static_cast<int>(__ldg(p.fills + static_cast<int64_t>(r) * p.fill_rs + e))
                      : min(p.bs, L - e * p.bs);
  }
}

__device__ __forceinline__ void walk_init(const PrefillParams &p, int r, int L, ChunkWalk &w) {
  w.e = 0;
  w.F = 0;
  w.E = p.fills ? __ldg(p.nent + r) : (L + p.bs - 1) / p.bs;
  w.have = false;
  walk_window(p, r, L, w, 0);
}

__device__ __forceinline__ bool walk_next(const PrefillParams &p, int r, int L, int pos_max,
                                          ChunkWalk &w, int &lo, int &hi, int &tb) {
  constexpr unsigned FULL = 0xffffffffu;
  const int bs = p.bs;
  while (w.e < w.E && w.F <= pos_max) {
    if (!w.have) {
      if (w.e - w.wb >= 32) walk_window(p, r, L, w, w.e);
      const int idx = w.e - w.wb;
      w.blk = __shfl_sync(FULL, w.wblk, idx);
      w.dir = __shfl_sync(FULL, w.wdir, idx);
      w.fill = __shfl_sync(FULL, w.wfill, idx);
      w.c = 0;
      w.have = true;
    }
    const int lo_s = w.dir ? bs - w.fill : 0, hi_s = w.dir ? bs : w.fill;
    while (w.c < bs / 16) {
      const int c = w.c++;
      lo = max(lo_s - 16 * c, 0);
      hi = min(hi_s - 16 * c, 16);
      if (lo >= hi) continue;
      tb = w.dir ? w.F + bs - 1 - 16 * c : w.F + 16 * c;   // token of chunk slot 0
      const int first_tok = w.dir ? tb - (hi - 1) : tb + lo;
      if (first_tok > pos_max) continue;
      return true;
    }
    w.F += w.fill;
    ++w.e;
    w.have = false;
  }
  return false;
}

}  // namespace

template <int D>
__global__ void __launch_bounds__(32 * (kConsumerWarps + 1), 1)
    prefill_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                   const PrefillParams p) {
  constexpr int HALF_BYTES = 16 * 128;
  constexpr int KV_BYTES = (D / 64) * HALF_BYTES;
  constexpr int SLOT_BYTES = 2 * KV_BYTES;
  constexpr int MT = D / 16;   // k-steps of Q.K^T, pairs of 8-wide d tiles of P.V
  // a PDL-launched successor (the mixed dispatch's decode kernel, which reads
  // nothing this kernel writes) may take SMs as this grid's CTAs finish
  asm volatile("griddepcontrol.launch_dependents;");
  constexpr unsigned FULL = 0xffffffffu;

  const int r = blockIdx.z, h = blockIdx.y;
  const int q0 = __ldg(p.cu_q + r);
  const int n = __ldg(p.cu_q + r + 1) - q0;
  const int g = p.g;
  const int rows = n * g;
  const int ntiles = (rows + kRowsPerTile - 1) / kRowsPerTile;
  const int tile = ntiles - 1 - static_cast<int>(blockIdx.x);   // longest (latest) tiles first
  if (tile < 0) return;
  const int L = __ldg(p.seq_lens + r);
  const int row0 = tile * kRowsPerTile;
  const int row_end = min(rows, row0 + kRowsPerTile);
  const int pos_max = L - n + (row_end - 1) / g;

  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t *gbase = smem_raw + (base - raw);
  int4 *metas = reinterpret_cast<int4 *>(gbase + kStages * SLOT_BYTES);     // per-stage chunk metadata
  uint64_t *bars = reinterpret_cast<uint64_t *>(metas + kStages);          // full[S], empty[S]
  const uint32_t full0 = smem_u32(bars), empty0 = full0 + 8 * kStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmK);
    prefetch_tmap(&tmV);
    for (int i = 0; i < kStages; ++i) {
      mbar_init(full0 + 8 * i, 1);
      mbar_init(empty0 + 8 * i, kConsumerWarps);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == kConsumerWarps) {
    ChunkWalk walk;
    walk_init(p, r, L, walk);
    int lo, hi, tb;
    // ------------------------------------------------------------ producer
    // Each stage's chunk metadata is handed over through named barrier
    // 1 + stage (producer bar.arrive, consumers bar.sync: release/acquire at
    // CTA scope); the tiles themselves complete on the stage's full mbarrier.
    const uint64_t pol = policy_evict_last();   // every query tile of the request re-reads these
    int it = 0;
    for (; walk_next(p, r, L, pos_max, walk, lo, hi, tb); ++it) {
      const int st = it % kStages;
      if (lane == 0) {
        const int round = it / kStages;
        if (round > 0) mbar_wait(empty0 + 8 * st, (round - 1) & 1);
        metas[st] = make_int4(lo, hi, tb, walk.dir);
        const uint32_t fb = full0 + 8 * st;
        mbar_arrive_expect_tx(fb, SLOT_BYTES);
        const uint32_t dk = base + st * SLOT_BYTES;
        const int c = walk.c - 1;
        tma_load_5d(dk, &tmK, 0, 16 * c, 0, h, walk.blk, fb, pol);
        tma_load_5d(dk + KV_BYTES, &tmV, 0, 16 * c, 0, h, walk.blk, fb, pol);
      }
      __syncwarp();
      named_bar_arrive(1 + st, 32 * (kConsumerWarps + 1));
    }
    const int st = it % kStages;   // terminator stage: metadata only
    if (lane == 0) {
      const int round = it / kStages;
      if (round > 0) mbar_wait(empty0 + 8 * st, (round - 1) & 1);
      metas[st] = make_int4(0, 0, 0, kLast);
    }
    __syncwarp();
    named_bar_arrive(1 + st, 32 * (kConsumerWarps + 1));
    return;
  }

  // ------------------------------------------------------------ consumers
  if (row0 + 16 * warp >= row_end) {   // no live rows in this warp (short tile, decode rows):
    for (int it = 0;; ++it) {          // keep the ring moving, skip the math
      const int st = it % kStages;
      named_bar_sync(1 + st, 32 * (kConsumerWarps + 1));
      if (metas[st].w & kLast) return;
      mbar_wait(full0 + 8 * st, (it / kStages) & 1);
      __syncwarp();
      if (lane == 0) mbar_arrive(empty0 + 8 * st);
    }
  }
  const int rA = row0 + 16 * warp + (lane >> 2), rB = rA + 8;
  // earliest query position of this warp's rows (rows are in position order)
  const int pos_warp_min = L - n + (row0 + 16 * warp) / g;
  const bool okA = rA < row_end, okB = rB < row_end;
  const int posA = okA ? L - n + rA / g : -1, posB = okB ? L - n + rB / g : -1;
  auto qrow = [&](int row) {
    const int tok = row / g, j = row - tok * g;
    return reinterpret_cast<const uint32_t *>(p.q + static_cast<int64_t>(q0 + tok) * p.q_st +
                                              static_cast<int64_t>(h * g + j) * p.q_sh);
  };
  const uint32_t *qa_ptr = qrow(okA ? rA : row0);
  const uint32_t *qb_ptr = qrow(okB ? rB : row0);
  uint32_t qf[MT][4];
#pragma unroll
  for (int ks = 0; ks < MT; ++ks) {
    const int c = ks * 8 + (lane & 3);   // 32-bit word = 2 bf16 at d = 2c
    qf[ks][0] = okA ? __ldg(qa_ptr + c) : 0u;
    qf[ks][1] = okB ? __ldg(qb_ptr + c) : 0u;
    qf[ks][2] = okA ? __ldg(qa_ptr + c + 4) : 0u;
    qf[ks][3] = okB ? __ldg(qb_ptr + c + 4) : 0u;
  }
  float oacc[2 * MT][4];
#pragma unroll
  for (int i = 0; i < 2 * MT; ++i) oacc[i][0] = oacc[i][1] = oacc[i][2] = oacc[i][3] = 0.f;
  float mA = -INFINITY, mB = -INFINITY, lA = 0.f, lB = 0.f;
  const int mi = lane >> 3, k0 = (lane & 3) * 2;

  for (int it = 0;; ++it) {
    const int st = it % kStages;
    named_bar_sync(1 + st, 32 * (kConsumerWarps + 1));
    const int4 meta = metas[st];
    if (meta.w & kLast) break;
    mbar_wait(full0 + 8 * st, (it / kStages) & 1);
    const int lo = meta.x, hi = meta.y, tb = meta.z, dir = meta.w;
    const uint32_t sk = base + st * SLOT_BYTES, sv = sk + KV_BYTES;
    // ---- S = Q.K^T (16 rows x 16 slots)
    float s0[4] = {0.f, 0.f, 0.f, 0.f}, s1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int ks = 0; ks < MT; ++ks) {
      const int tok = (mi >> 1) * 8 + (lane & 7), de = ks * 16 + (mi & 1) * 8;
      uint32_t b00, b01, b10, b11;
      ldsm_x4(sk + (de >> 6) * HALF_BYTES + pswz(tok, (de & 63) >> 3), b00, b01, b10, b11);
      mma_bf16_16816(s0, qf[ks][0], qf[ks][1], qf[ks][2], qf[ks][3], b00, b01);
      mma_bf16_16816(s1, qf[ks][0], qf[ks][1], qf[ks][2], qf[ks][3], b10, b11);
    }
    // ---- direction + causal mask by token index, scale to the log2 domain
    float sv4[2][4] = {{s0[0], s0[1], s0[2], s0[3]}, {s1[0], s1[1], s1[2], s1[3]}};
    const int max_tok = dir ? tb - lo : tb + hi - 1;
    if (lo == 0 && hi == 16 && max_tok <= pos_warp_min) {   // whole chunk visible to every row
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) sv4[nt][e] *= p.scale_log2;
    } else {
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int col = nt * 8 + k0 + (e & 1);
          const int tok = dir ? tb - col : tb + col;
          const bool ok = col >= lo && col < hi && tok <= ((e >> 1) ? posB : posA);
          sv4[nt][e] = ok ? sv4[nt][e] * p.scale_log2 : -INFINITY;
        }
    }
    float mxA = fmaxf(fmaxf(sv4[0][0], sv4[0][1]), fmaxf(sv4[1][0], sv4[1][1]));
    float mxB = fmaxf(fmaxf(sv4[0][2], sv4[0][3]), fmaxf(sv4[1][2], sv4[1][3]));
    mxA = fmaxf(mxA, __shfl_xor_sync(FULL, mxA, 1));
    mxA = fmaxf(mxA, __shfl_xor_sync(FULL, mxA, 2));
    mxB = fmaxf(mxB, __shfl_xor_sync(FULL, mxB, 1));
    mxB = fmaxf(mxB, __shfl_xor_sync(FULL, mxB, 2));
    const float mnA = fmaxf(mA, mxA), mnB = fmaxf(mB, mxB);
    const float gA = mnA == -INFINITY ? 0.f : mnA, gB = mnB == -INFINITY ? 0.f : mnB;
    const float alA = ex2(mA - gA), alB = ex2(mB - gB);
    float pr[2][4];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      pr[nt][0] = ex2(sv4[nt][0] - gA);
      pr[nt][1] = ex2(sv4[nt][1] - gA);
      pr[nt][2] = ex2(sv4[nt][2] - gB);
      pr[nt][3] = ex2(sv4[nt][3] - gB);
    }
    lA = lA * alA + (pr[0][0] + pr[0][1]) + (pr[1][0] + pr[1][1]);
    lB = lB * alB + (pr[0][2] + pr[0][3]) + (pr[1][2] + pr[1][3]);
    mA = mnA;
    mB = mnB;
    if (alA != 1.f || alB != 1.f) {
#pragma unroll
      for (int i = 0; i < 2 * MT; ++i) {
        oacc[i][0] *= alA;
        oacc[i][1] *= alA;
        oacc[i][2] *= alB;
        oacc[i][3] *= alB;
      }
    }
    // ---- O += P.V (P from the S accumulators; dead V rows masked to zero)
    const uint32_t pa0 = pack_bf16(pr[0][0], pr[0][1]), pa1 = pack_bf16(pr[0][2], pr[0][3]);
    const uint32_t pa2 = pack_bf16(pr[1][0], pr[1][1]), pa3 = pack_bf16(pr[1][2], pr[1][3]);
    auto live = [&](int s) { return s >= lo && s < hi; };
    const uint32_t vm0 = (live(k0) ? 0x0000FFFFu : 0u) | (live(k0 + 1) ? 0xFFFF0000u : 0u);
    const uint32_t vm1 = (live(k0 + 8) ? 0x0000FFFFu : 0u) | (live(k0 + 9) ? 0xFFFF0000u : 0u);
#pragma unroll
    for (int dt2 = 0; dt2 < MT; ++dt2) {
      const int tok = (mi & 1) * 8 + (lane & 7), de = dt2 * 16 + (mi >> 1) * 8;
      uint32_t v0, v1, v2, v3;
      ldsm_x4_t(sv + (de >> 6) * HALF_BYTES + pswz(tok, (de & 63) >> 3), v0, v1, v2, v3);
      mma_bf16_16816(oacc[2 * dt2], pa0, pa1, pa2, pa3, v0 & vm0, v1 & vm1);
      mma_bf16_16816(oacc[2 * dt2 + 1], pa0, pa1, pa2, pa3, v2 & vm0, v3 & vm1);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * st);
  }
  // ---- epilogue: normalise, round to bf16 (RNE), write the valid rows
  lA += __shfl_xor_sync(FULL, lA, 1);
  lA += __shfl_xor_sync(FULL, lA, 2);
  lB += __shfl_xor_sync(FULL, lB, 1);
  lB += __shfl_xor_sync(FULL, lB, 2);
  const float iA = lA > 0.f ? 1.f / lA : 0.f, iB = lB > 0.f ? 1.f / lB : 0.f;
  auto orow = [&](int row) {
    const int tok = row / g, j = row - tok * g;
    return reinterpret_cast<uint32_t *>(p.out + static_cast<int64_t>(q0 + tok) * p.o_st +
                                        static_cast<int64_t>(h * g + j) * p.o_sh);
  };
  if (okA) {
    uint32_t *o = orow(rA);
#pragma unroll
    for (int i = 0; i < 2 * MT; ++i) o[i * 4 + (lane & 3)] = pack_bf16(oacc[i][0] * iA, oacc[i][1] * iA);
  }
  if (okB) {
    uint32_t *o = orow(rB);
#pragma unroll
    for (int i = 0; i < 2 * MT; ++i) o[i * 4 + (lane & 3)] = pack_bf16(oacc[i][2] * iB, oacc[i][3] * iB);
  }
}

// head_dim 128 runs the tcgen05/TMEM kernel (prefill_tc.cu): Llama-70B TP1 whole-
// prompt prefills 160 vs 140 TF/s for this mma.sync kernel, which stays the
// head_dim-64 path and is selectable for 128 with BKV_PREFILL_MMA_SYNC=1 (dev A/B).
bool prefill_uses_tc(int head_dim) {
  return head_dim == 128 && dev_switches().prefill_mma_sync == 0;
}

int prefill_smem_bytes(int head_dim) {
  return 1024 + kStages * 2 * (head_dim / 64) * 2048 + kStages * 16 + 2 * kStages * 8;
}

template <int D>
static cudaError_t launch_prefill_t(const CUtensorMap &tmK, const CUtensorMap &tmV,
                                    const PrefillParams &p, int max_q_len, cudaStream_t s) {
  const int smem = prefill_smem_bytes(D);
  {
    cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void *>(prefill_kernel<D>), smem);
    if (e != cudaSuccess) return e;
  }
  const long long tiles = (static_cast<long long>(max_q_len) * p.g + kRowsPerTile - 1) / kRowsPerTile;
  dim3 grid(static_cast<unsigned>(tiles), p.H, p.B);
  prefill_kernel<D><<<grid, 32 * (kConsumerWarps + 1), smem, s>>>(tmK, tmV, p);
  return cudaGetLastError();
}

cudaError_t launch_prefill(const CUtensorMap &tmK, const CUtensorMap &tmV, const CUtensorMap *tmQ,
                           const CUtensorMap *tmO, const PrefillParams &p, int head_dim, int max_q_len, cudaStream_t s) {
  if (p.B <= 0 || max_q_len <= 0) return cudaSuccess;
  // head_dim 128: the tcgen05 / TMEM kernel (prefill_tc.cu; tensor maps with one 64-d half per box)
  if (prefill_uses_tc(head_dim)) return launch_prefill_tc(tmK, tmV, tmQ, tmO, p, max_q_len, s);
  return head_dim == 128 ? launch_prefill_t<128>(tmK, tmV, p, max_q_len, s)
                         : launch_prefill_t<64>(tmK, tmV, p, max_q_len, s);
}

}  // namespace bkv
