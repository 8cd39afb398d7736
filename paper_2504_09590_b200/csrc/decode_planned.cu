// decode_planned.cu -- paged decode attention over BROS's bidirectional KV
// cache with a HOST-BUILT static split plan and the split merge inside the
// kernel: one launch per layer (PAPER.md
// P:711).
//
// What it computes is the same as decode_attention.cu (reading of SURVEY §8(c)
// step 5): for request r, q head h, kv head h/g,
//     out = softmax_t(scale * q.K_t) . V_t   over the resident tokens t < L_r,
// read through the block table and the same-shaped direction table; a forward
// (RT) entry holds its tokens in slots [0, n), a reversed (BE) entry in
// [bs-n, bs).  Attention is a sum over the token SET, so blocks are
// consumed in physical slot order and the direction only selects live slots.
//
// Why a second kernel (DESIGN.md §6 "planned decode"): the small head shards of
// tensor parallelism (Llama-2-70B TP8: 77 MB per layer, 12 us at the HBM
// copy peak) are bounded by fixed costs of the dynamically scheduled kernel --
// an in-kernel split-plan prologue (~3 us), unit-size imbalance at the tail
// (~2.5 us) and a second, stream-ordered merge launch (~3 us).  Here:
//  * the plan (decode_plan.cu) comes from the host once per step: every warp
//    streams an equal contiguous range of the flattened (request, kv head,
//    block) sequence, so all warps finish together;
//  * the plan, lengths and block-table windows are read before the PDL grid
//    wait, so a layer starts streaming as soon as the previous one completes;
//  * the resident KV of the warp's first entries is requested (ring tiles) or
//    prefetched into L2 before the PDL grid wait, while the previous kernel
//    drains (BKV_FLAG_KV_EARLY);
//  * rows cut across the warps of a CTA are merged from shared memory after
//    the CTA's last block; rows cut across CTAs leave one combined piece per
//    CTA in the workspace, merged by planned_xmerge_kernel, the next kernel on
//    the stream (no thread ever waits for another CTA: no deadlock whatever
//    the residency).
// The streaming core is the one of decode_kernel: per-warp 2-deep rings of
// 128B-swizzled smem slots filled by ONE 5-D TMA box per 16-slot chunk (K and
// V of one (block, kv head)), mbarrier completion, S^T = K.Q^T and
// O^T += V^T.P^T on bf16 mma.sync with tokens on M (every group size), the
// fused append of this step's token (bkv_decode_step semantics), dead slots
// selected to -inf and their V rows zeroed (reading Q10).
#include <math.h>
#include <stddef.h>

#include "bkv_internal.h"
#include "bkv_ptx.cuh"

namespace bkv {
namespace planned {

#ifdef BKV_DEV_TRACE
constexpr bool kTrace = true;   // dev timeline stamps (scripts/trace_planned.py)
#else
constexpr bool kTrace = false;
#endif

enum : int { F_FIRST = 1, F_LAST = 2, F_NOKV = 4, F_NEW = 16 };

struct SlotMeta {   // 32 bytes: one ring slot's chunk
  int seg, r, h, split;
  int lo, hi, flags, aux;
};

template <int D>
struct Geo {
  static constexpr int HALVES = D / 64;
  static constexpr int HALF_BYTES = 16 * 128;
  static constexpr int KV_BYTES = HALVES * HALF_BYTES;
  static constexpr int SLOT_BYTES = 2 * KV_BYTES;
};

__device__ __forceinline__ uint32_t swz(int row, int c) {
  return static_cast<uint32_t>(row * 128 + ((c ^ (row & 7)) << 4));
}

// shared-memory bytes of one warp's piece (m, l, o of its g rows), g <= gmax
__host__ __device__ constexpr int piece_bytes(int D, int gmax) { return gmax * (D + 2) * 4; }
// floats per global piece slot: o[g][D], then (m, l)[g], padded to 16 bytes
__host__ __device__ constexpr int piece_stride(int g, int D) { return (g * (D + 2) + 3) & ~3; }

struct WarpSmem {   // byte offsets inside one warp's region
  int ring, metas, bars, scr, patch, piece, total;
};
__host__ __device__ inline WarpSmem warp_smem(int D, int gmax, int S) {
  WarpSmem w;
  const int slot = 2 * (D / 64) * 2048;   // K and V tiles of one 16-slot chunk
  const int ring = S * slot > piece_bytes(D, gmax) ? S * slot : piece_bytes(D, gmax);   // also piece slot 1
  w.ring = 0;
  w.metas = ring;
  w.bars = w.metas + S * 32;
  w.scr = (w.bars + S * 8 + 127) & ~127;
  w.patch = w.scr + 1024;
  w.piece = w.patch + S * 512;
  w.total = (w.piece + piece_bytes(D, gmax) + 1023) & ~1023;
  return w;
}

// 1/x for a softmax denominator (x >= 1 whenever a token is live: the maximum
// contributes ex2(0)), 0 for an empty row; MUFU reciprocal, no IEEE slow path.
__device__ __forceinline__ float rcp_pos(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return x > 0.f ? r : 0.f;
}

template <int D, bool G16>
__global__ void __launch_bounds__(256, 1)
    planned_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                   const PlannedParams p) {
  using G = Geo<D>;
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int GMAX = G16 ? 16 : 8;
  constexpr int NT = G16 ? 2 : 1;
  constexpr int MT = D / 16;
  constexpr int EPL = D / 32;

  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const int W = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = p.slots;
  const WarpSmem ws = warp_smem(D, GMAX, S);
  const uint32_t wbase = base + warp * ws.total;
  const uint32_t my_slots = wbase + ws.ring, my_bars = wbase + ws.bars, my_scr = wbase + ws.scr;
  const uint32_t my_patch = wbase + ws.patch;
  uint8_t *gw_ptr = smem_raw + (base - raw) + warp * ws.total;
  SlotMeta *metas = reinterpret_cast<SlotMeta *>(gw_ptr + ws.metas);
  const int g = p.g, H = p.H, bs = p.bs;
  const int chunks_per_block = bs >> 4;
  const int gw = blockIdx.x * W + warp;

  // dev trace: stamp k of this warp (0 entry, 1 pre-wait reads, 2 grid wait, 3 first tile,
  // 4 streaming done, 5 CTA barrier, 6 merges done)
  auto stamp = [&](int k) {
    if (kTrace && p.trace != nullptr && lane == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      p.trace[(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 16 + k] = t;
    }
  };
  stamp(0);
  if (threadIdx.x == 0) {
    prefetch_tmap(&tmK);
    prefetch_tmap(&tmV);
  }
  if (p.pdl) asm volatile("griddepcontrol.launch_dependents;");

  // ---------------------------------------------------------- pre-wait reads
  // The plan is step metadata (BKV_FLAG_PDL contract: not written by the
  // immediately preceding kernel), so it is read while that kernel drains.  It
  // carries the step's block map already flattened in warp order: warp w's
  // blocks are entries [w P, w P + n) of the packed entry list (block id,
  // direction, live tokens, last-entry bit), so the first TMA needs ONE
  // dependent load, issued together with the segment descriptors.
  const int P = __ldg(p.plan_hdr + offsetof(PlanHeader, P) / 4);
  const int s0 = __ldg(p.wseg + gw), s1 = __ldg(p.wseg + gw + 1);
  const int ent0 = gw * P;                          // the warp's first flattened entry
  const int n_mine = min(P, __ldg(p.plan_hdr + offsetof(PlanHeader, total) / 4) - ent0);   // its entries
  int4 sg_l = make_int4(0, 0, 0, 0);
  auto load_segs = [&](int first) {
    const int si = first + lane;
    if (si < s1) sg_l = __ldg(p.segs + 2 * si);
  };
  int seg_base = s0;
  load_segs(seg_base);
  uint32_t ent_w = 0;                               // lane i: packed entry ent0 + ent_base + i
  int ent_base = 0;
  auto load_ents = [&](int first) {
    ent_base = first;
    if (first + lane < n_mine) ent_w = __ldg(p.ent + ent0 + first + lane);
  };
  load_ents(0);

  struct SegInfo {
    int si, r, h, e0, e1, split;
  };
  auto seg_info = [&](int si) -> SegInfo {
    SegInfo x;
    x.si = si;
    if (si >= s1) return x;
    if (si - seg_base >= 32) {   // more than 32 segments in this warp's range (short rows)
      seg_base = si;
      load_segs(seg_base);
    }
    const int j = si - seg_base;
    x.r = __shfl_sync(FULL, sg_l.x, j);
    x.h = __shfl_sync(FULL, sg_l.y, j);
    x.e0 = __shfl_sync(FULL, sg_l.z, j);
    const int w4 = __shfl_sync(FULL, sg_l.w, j);
    x.e1 = w4 & 0xffff;
    x.split = (w4 >> kPlanSplitBit) & 1;
    return x;
  };
  const int n_zero = __ldg(p.plan_hdr + offsetof(PlanHeader, n_zero) / 4);   // plan data: pre-wait
  // this CTA's merge tasks (<= 2 per warp: a warp has at most two split segments)
  __shared__ int4 task_s[2 * 2 * kPlannedWarps];
  const int t_beg = __ldg(p.ctask + blockIdx.x), t_end = __ldg(p.ctask + blockIdx.x + 1);
  if (threadIdx.x < 2 * (t_end - t_beg)) task_s[threadIdx.x] = __ldg(p.tasks + 2 * t_beg + threadIdx.x);
  SegInfo cur{}, nxt = seg_info(s0);

  // L2 prefetch of the warp's next entries (BKV_FLAG_KV_EARLY contract: the
  // resident KV is not written by the preceding kernel).  The ring's own first
  // tiles are requested below; lane k hints entry k < pf of the range, so the
  // HBM, idle while the previous kernel drains, already streams this layer.
  if (p.kv_early && p.pf > 0) {
    const int npf = min(p.pf, n_mine), skip = S / chunks_per_block;
    int my_h = 0;
    for (int j = 0, k0 = 0; k0 < npf && s0 + j < s1 && j < 32; ++j) {   // head of entry `lane`
      const int h = __shfl_sync(FULL, sg_l.y, j);
      const int len = (__shfl_sync(FULL, sg_l.w, j) & 0xffff) - __shfl_sync(FULL, sg_l.z, j);
      if (lane >= k0 && lane < k0 + len) my_h = h;
      k0 += len;
    }
    if (lane >= skip && lane < npf) {
      const int b = static_cast<int>(ent_w & kEntBlockMask);
      const int dr = (ent_w >> kEntDirShift) & 1;
      const int ne = static_cast<int>((ent_w >> kEntFillShift) & 31u) + 1;
      const int lo_s = dr ? bs - ne : 0, hi_s = dr ? bs : ne;
      for (int c = 0; c < chunks_per_block; ++c) {
        if (min(hi_s - c * 16, 16) <= max(lo_s - c * 16, 0)) continue;   // no live slot in this chunk
        if (p.kv_mode) {
          tma_prefetch_5d(&tmK, 0, c * 16, 0, 0, b * H + my_h);
        } else {
          tma_prefetch_5d(&tmK, 0, c * 16, 0, my_h, b);
          tma_prefetch_5d(&tmV, 0, c * 16, 0, my_h, b);
        }
      }
    }
  }

  if (kTrace) {   // (the stamp needs the loads to have landed)
    volatile int sink = static_cast<int>(ent_w) + nxt.r;
    (void)sink;
    stamp(1);
  }
  if (lane == 0) {
    for (int i = 0; i < S; ++i) mbar_init(my_bars + 8 * i, 1);
    fence_mbar_init();
  }
  __syncwarp();
  const uint64_t pol = policy_evict_first();
  // Everything after the grid wait may touch data the preceding kernel wrote (q,
  // k_new, the workspace of the previous call).  BKV_FLAG_KV_EARLY: the resident
  // KV is not written by that kernel, so the ring's first tiles are requested
  // before the wait (a new-token chunk, which reads k_new/v_new, waits first).
  bool waited = !p.pdl;
  auto grid_wait = [&]() {
    if (!waited) {
      asm volatile("griddepcontrol.wait;" ::: "memory");
      waited = true;
      stamp(2);
    }
  };
  if (!p.kv_early) grid_wait();

  bool is_active = false, is_done = false, is_first = false;
  int is_ci = 0, is_nc = 0, ent_pos = 0;
  // next chunk of the warp's stream: 16 slots (sub-chunk ci % cpb) of entry e0 + ci / cpb
  auto next_chunk = [&](SlotMeta &m, int &blk, int &csub) -> bool {
    if (!is_active) {
      if (is_done || nxt.si >= s1) {
        is_done = true;
        return false;
      }
      cur = nxt;
      nxt = seg_info(cur.si + 1);
      if (lane < g) {   // the segment's q rows into L2 (read by the consumer later)
        const uint16_t *qrow = p.q + static_cast<int64_t>(cur.r) * p.q_ss +
                               static_cast<int64_t>(cur.h * g + lane) * p.q_sh;
        asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(qrow));
        if (D == 128) asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(qrow + 64));
      }
      is_ci = 0;
      is_nc = (cur.e1 - cur.e0) * chunks_per_block;
      is_first = true;
      is_active = true;
    }
    const int k = ent_pos + (chunks_per_block == 1 ? is_ci : (is_ci >> 1));   // entry within the warp range
    const int c = chunks_per_block == 1 ? 0 : (is_ci & 1);
    if (k - ent_base >= 32) load_ents(k);
    const uint32_t en = __shfl_sync(FULL, ent_w, k - ent_base);
    const int b = static_cast<int>(en & kEntBlockMask);
    const int dr = (en >> kEntDirShift) & 1;
    const int ne = static_cast<int>((en >> kEntFillShift) & 31u) + 1;   // live tokens of the entry
    const int lo_s = dr ? bs - ne : 0;                                 // RT from the left,
    const int hi_s = dr ? bs : ne;                                     //        BE from the right
    const int lo = max(lo_s - c * 16, 0), hi = min(hi_s - c * 16, 16);
    int flags = (is_first ? F_FIRST : 0) | (lo >= hi ? F_NOKV : 0);
    if (p.k_new != nullptr && (en >> kEntLastShift)) {   // fused step: token L-1 lives in the last entry
      const int j = ne - 1;
      const int slot_new = dr ? bs - 1 - j : j;
      if ((slot_new >> 4) == c) flags |= F_NEW | (slot_new << 8);
    }
    is_first = false;
    csub = c;
    blk = b;
    is_ci += 1;
    if (is_ci >= is_nc) {
      flags |= F_LAST;
      is_active = false;
      ent_pos += cur.e1 - cur.e0;
    }
    m = SlotMeta{cur.si, cur.r, cur.h, cur.split, lo, hi, flags, b};
    return true;
  };

  auto issue = [&](int i, const SlotMeta &m, int blk, int csub) {
    if (lane == 0) {
      reinterpret_cast<int4 *>(metas + i)[0] = make_int4(m.seg, m.r, m.h, m.split);
      reinterpret_cast<int4 *>(metas + i)[1] = make_int4(m.lo, m.hi, m.flags, m.aux);
      const uint32_t bar = my_bars + 8 * i;
      const bool kv = !(m.flags & F_NOKV);
      const bool nw = m.flags & F_NEW;
      mbar_arrive_expect_tx(bar, (kv ? G::SLOT_BYTES : 0) + (nw ? 4 * D : 0));
      if (nw) {
        bulk_wait_read_all();   // the previous bulk store out of the patch area has read it
        const int64_t row = (static_cast<int64_t>(m.r) * H + m.h) * D;
        bulk_load(my_patch + i * 512, p.k_new + row, 2 * D, bar);
        bulk_load(my_patch + i * 512 + 2 * D, p.v_new + row, 2 * D, bar);
      }
      if (kv) {
        const uint32_t dk = my_slots + i * G::SLOT_BYTES, dv = dk + G::KV_BYTES;
        if (p.kv_mode) {
          tma_load_5d(dk, &tmK, 0, csub * 16, 0, 0, blk * H + m.h, bar, pol);
        } else {
          tma_load_5d(dk, &tmK, 0, csub * 16, 0, m.h, blk, bar, pol);
          tma_load_5d(dv, &tmV, 0, csub * 16, 0, m.h, blk, bar, pol);
        }
      }
    }
  };

  // ------------------------------------------------------------- consumer
  uint32_t qb[MT][NT][2];
  float oacc[MT][NT][4];
  float mrun[NT][2], lrun[NT][2];
  auto begin_seg = [&](const SlotMeta &m) {
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      mrun[n][0] = mrun[n][1] = -INFINITY;
      lrun[n][0] = lrun[n][1] = 0.f;
    }
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int n = 0; n < NT; ++n) oacc[mt][n][0] = oacc[mt][n][1] = oacc[mt][n][2] = oacc[mt][n][3] = 0.f;
    const uint16_t *qg = p.q + static_cast<int64_t>(m.r) * p.q_ss + static_cast<int64_t>(m.h * g) * p.q_sh;
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const int head = n * 8 + (lane >> 2);
      const bool ok = head < g;
      const uint32_t *qh = reinterpret_cast<const uint32_t *>(qg + static_cast<int64_t>(ok ? head : 0) * p.q_sh) + (lane & 3);
#pragma unroll
      for (int ks = 0; ks < MT; ++ks) {
        qb[ks][n][0] = ok ? __ldg(qh + ks * 8) : 0u;
        qb[ks][n][1] = ok ? __ldg(qh + ks * 8 + 4) : 0u;
      }
    }
  };
  auto zero_dead_rows = [&](uint32_t sv, int lo, int hi) {
    for (int idx = lane; idx < 16 * G::HALVES * 8; idx += 32) {
      const int row = idx / (G::HALVES * 8), rest = idx - row * (G::HALVES * 8);
      if (row < lo || row >= hi) sts128_zero(sv + (rest >> 3) * G::HALF_BYTES + row * 128 + (rest & 7) * 16);
    }
    __syncwarp();
  };
  const uint32_t k_off = p.kv_mode == 2 ? G::KV_BYTES : 0u, v_off = G::KV_BYTES - k_off;
  auto consume = [&](uint32_t s0a, int lo, int hi, auto &&release) {
    const uint32_t sk = s0a + k_off, sv = s0a + v_off;
    if (lo > 0 || hi < 16) zero_dead_rows(sv, lo, hi);   // P = 0 must never meet NaN (Q10)
    const int mi = lane >> 3;
    float sa[NT][4], sb[NT][4];
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
      for (int j = 0; j < 4; ++j) sa[n][j] = sb[n][j] = 0.f;
#pragma unroll
    for (int ks = 0; ks < MT; ++ks) {   // S^T = K . Q^T: 16 tokens x 8 heads per n tile
      const int tok = (mi & 1) * 8 + (lane & 7), de = ks * 16 + (mi >> 1) * 8;
      uint32_t a0, a1, a2, a3;
      ldsm_x4(sk + (de >> 6) * G::HALF_BYTES + swz(tok, (de & 63) >> 3), a0, a1, a2, a3);
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        float(&acc)[4] = (ks & 1) ? sb[n] : sa[n];
        mma_bf16_16816(acc, a0, a1, a2, a3, qb[ks][n][0], qb[ks][n][1]);
      }
    }
    uint32_t va[MT][4];   // A = V^T via ldmatrix.trans, then the slot is free
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int tok = (mi >> 1) * 8 + (lane & 7), de = mt * 16 + (mi & 1) * 8;
      ldsm_x4_t(sv + (de >> 6) * G::HALF_BYTES + swz(tok, (de & 63) >> 3), va[mt][0], va[mt][1], va[mt][2],
                va[mt][3]);
    }
    release();
    const int t0 = lane >> 2, t1 = t0 + 8;
    const bool ok0 = t0 >= lo && t0 < hi, ok1 = t1 >= lo && t1 < hi;
    // Lazy reference maximum (log2 domain): the common chunk takes the running
    // reference mrun as its exponent base (p <= 2^8); only when a live score passes
    // it by more than 8 does the warp reduce the chunk's exact maximum across lanes
    // and rescale l and O (the first chunk of a segment, and rarely after): the
    // shuffles, the correction exponential and the O rescale leave the common path.
    float sv0[NT][2], sv1[NT][2];
    bool need = false;
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        sv0[n][j] = ok0 ? (sa[n][j] + sb[n][j]) * p.scale_log2 : -INFINITY;
        sv1[n][j] = ok1 ? (sa[n][2 + j] + sb[n][2 + j]) * p.scale_log2 : -INFINITY;
        need |= fmaxf(sv0[n][j], sv1[n][j]) > mrun[n][j] + 8.f;
      }
    if (__any_sync(FULL, need)) {
      float alpha[NT][2];
#pragma unroll
      for (int n = 0; n < NT; ++n)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          float mx = fmaxf(sv0[n][j], sv1[n][j]);
          mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, 4));
          mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, 8));
          mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, 16));
          const float mnew = fmaxf(mrun[n][j], mx);
          alpha[n][j] = mnew == -INFINITY ? 1.f : ex2(mrun[n][j] - mnew);   // mrun = -inf: 0
          lrun[n][j] *= alpha[n][j];
          mrun[n][j] = mnew;
        }
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          const float2 a2 = make_float2(alpha[n][0], alpha[n][1]);
          const float2 lo2 = __fmul2_rn(make_float2(oacc[mt][n][0], oacc[mt][n][1]), a2);
          const float2 hi2 = __fmul2_rn(make_float2(oacc[mt][n][2], oacc[mt][n][3]), a2);
          oacc[mt][n][0] = lo2.x;
          oacc[mt][n][1] = lo2.y;
          oacc[mt][n][2] = hi2.x;
          oacc[mt][n][3] = hi2.y;
        }
    }
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const float base_m = mrun[n][j] == -INFINITY ? 0.f : mrun[n][j];   // no live token yet: p = 0
        const float p0 = ex2(sv0[n][j] - base_m), p1 = ex2(sv1[n][j] - base_m);
        lrun[n][j] += p0 + p1;
        const int head = n * 8 + (lane & 3) * 2 + j;   // P^T -> scratch as P[head][token]
        st_shared_bf16(my_scr + head * 48 + t0 * 2, p0);
        st_shared_bf16(my_scr + head * 48 + t1 * 2, p1);
      }
    __syncwarp();
    uint32_t pb[NT][2];
    if constexpr (NT == 1) {
      const int r8 = lane & 7, hi8 = (lane >> 3) & 1;
      ldsm_x2(my_scr + r8 * 48 + hi8 * 16, pb[0][0], pb[0][1]);
    } else {
      const int r8 = lane & 7, hi8 = (lane >> 3) & 1, nn = lane >> 4;
      ldsm_x4(my_scr + (nn * 8 + r8) * 48 + hi8 * 16, pb[0][0], pb[0][1], pb[1][0], pb[1][1]);
    }
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int n = 0; n < NT; ++n)
        mma_bf16_16816(oacc[mt][n], va[mt][0], va[mt][1], va[mt][2], va[mt][3], pb[n][0], pb[n][1]);
  };

  auto store_row = [&](int r, int head_global, const float *o, float inv) {
    // bf16 output row elements [lane*EPL, lane*EPL + EPL) (+ the fused reassembly's peers)
    const int64_t off = static_cast<int64_t>(r) * p.o_ss + static_cast<int64_t>(head_global) * p.o_sh + lane * EPL;
    if constexpr (EPL == 4) {
      uint2 w;
      w.x = pack_bf16(o[0] * inv, o[1] * inv);
      w.y = pack_bf16(o[2] * inv, o[3] * inv);
      *reinterpret_cast<uint2 *>(p.out + off) = w;
      peer_put8(p, off, w);
    } else {
      const uint32_t w = pack_bf16(o[0] * inv, o[1] * inv);
      *reinterpret_cast<uint32_t *>(p.out + off) = w;
      peer_put4(p, off, w);
    }
  };

  // piece layout (smem or global): o[head][D] fp32, then (m, l)[head]
  auto end_seg = [&](const SlotMeta &m) {
    float lsum[NT][2];
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        float l = lrun[n][j];
        l += __shfl_xor_sync(FULL, l, 4);
        l += __shfl_xor_sync(FULL, l, 8);
        l += __shfl_xor_sync(FULL, l, 16);
        lsum[n][j] = l;
      }
    const int d0 = lane >> 2;
    if (!m.split) {   // the whole row is this warp's: normalise and store bf16
#pragma unroll
      for (int n = 0; n < NT; ++n)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int head = n * 8 + (lane & 3) * 2 + j;
          if (head >= g) continue;
          const float inv = rcp_pos(lsum[n][j]);
          uint16_t *o = p.out + static_cast<int64_t>(m.r) * p.o_ss + static_cast<int64_t>(m.h * g + head) * p.o_sh;
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            const __nv_bfloat16 b0 = __float2bfloat16_rn(oacc[mt][n][j] * inv);
            const __nv_bfloat16 b1 = __float2bfloat16_rn(oacc[mt][n][2 + j] * inv);
            o[mt * 16 + d0] = *reinterpret_cast<const uint16_t *>(&b0);
            o[mt * 16 + d0 + 8] = *reinterpret_cast<const uint16_t *>(&b1);
          }
        }
      if (p.n_peers > 0) {   // fused reassembly: forward the rows to the peers with vector stores
        __syncwarp();
        for (int head = 0; head < g; ++head) {
          const int64_t off = static_cast<int64_t>(m.r) * p.o_ss + static_cast<int64_t>(m.h * g + head) * p.o_sh +
                              lane * EPL;
          if constexpr (EPL == 4) {
            const uint2 w = __ldcg(reinterpret_cast<const uint2 *>(p.out + off));
            peer_put8(p, off, w);
          } else {
            const uint32_t w = __ldcg(reinterpret_cast<const unsigned int *>(p.out + off));
            peer_put4(p, off, w);
          }
        }
      }
      return;
    }
    // split row: park (m, l, o) in this warp's piece slot -- slot 0 = the
    // dedicated area (the warp's first segment), slot 1 = the ring (the warp's
    // last segment: its streaming is over)
    const uint32_t pc = (m.seg == s0) ? wbase + ws.piece : my_slots;
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int head = n * 8 + (lane & 3) * 2 + j;
        if (head >= g) continue;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          st_shared_f32(pc + (head * D + mt * 16 + d0) * 4, oacc[mt][n][j]);
          st_shared_f32(pc + (head * D + mt * 16 + d0 + 8) * 4, oacc[mt][n][2 + j]);
        }
        if (d0 == 0) st_shared_v2f(pc + (g * D + 2 * head) * 4, mrun[n][j], lsum[n][j]);
      }
  };

  // ------------------------------------------------------------ main loop
  int issued = 0;
  for (; issued < S; ++issued) {
    SlotMeta m;
    int blk, cs;
    if (!next_chunk(m, blk, cs)) break;
    if (m.flags & F_NEW) grid_wait();
    issue(issued, m, blk, cs);
  }
  grid_wait();
  int slot = 0;
  uint32_t phase = 0;
  for (int seq = 0; seq < issued; ++seq) {
    __syncwarp();
    const int4 mw0 = reinterpret_cast<const int4 *>(metas + slot)[0];
    const int4 mw1 = reinterpret_cast<const int4 *>(metas + slot)[1];
    const SlotMeta m{mw0.x, mw0.y, mw0.z, mw0.w, mw1.x, mw1.y, mw1.z, mw1.w};
    mbar_wait(my_bars + 8 * slot, phase);
    if (kTrace && seq == 0) stamp(3);
    if (m.flags & F_FIRST) begin_seg(m);
    if (m.flags & F_NEW) {   // patch the new token's row into the tile and store it into the pool
      constexpr int TPR = D / 8;
      const int which = lane >> 4, pcx = lane & 15, slot_new = (m.flags >> 8) & 0xff;
      if (pcx < TPR) {
        const uint4 v = lds128(my_patch + slot * 512 + which * 2 * D + pcx * 16);
        const uint32_t tile = my_slots + slot * G::SLOT_BYTES + (which ? v_off : k_off);
        st_shared_v4(tile + (pcx >> 3) * G::HALF_BYTES + swz(slot_new & 15, pcx & 7), v);
      }
      if (lane == 0) {
        const int64_t off = static_cast<int64_t>(m.aux) * p.pool_sb + static_cast<int64_t>(m.h) * p.pool_sh +
                            static_cast<int64_t>(slot_new) * p.pool_ss;
        bulk_store(p.k_pool + off, my_patch + slot * 512, 2 * D);
        bulk_store(p.v_pool + off, my_patch + slot * 512 + 2 * D, 2 * D);
        bulk_commit();
      }
      __syncwarp();
    }
    auto release = [&]() {
      __syncwarp();
      if (m.lo > 0 || m.hi < 16 || (m.flags & F_NEW)) fence_proxy_async_smem();
      SlotMeta mn;
      int blk, cs;
      if (next_chunk(mn, blk, cs)) {
        issue(slot, mn, blk, cs);
        ++issued;
      }
    };
    if (!(m.flags & F_NOKV))
      consume(my_slots + slot * G::SLOT_BYTES, m.lo, m.hi, release);
    else
      release();
    if (m.flags & F_LAST) end_seg(m);
    if (++slot == S) {
      slot = 0;
      phase ^= 1u;
    }
  }
  if (p.k_new != nullptr && lane == 0) bulk_wait_all();   // pool rows written (and patch read) before exit
  stamp(4);

  // ------------------------------------------------ rows without tokens (Q8)
  {
    const int nw = gridDim.x * W;
    for (int z = gw; z < n_zero; z += nw) {
      const int r = __ldg(p.zero + 2 * z), h = __ldg(p.zero + 2 * z + 1);
      const float o0[EPL] = {};
      for (int head = 0; head < g; ++head) store_row(r, h * g + head, o0, 0.f);
    }
  }

  // ------------------------------------------------------ split merges (a5)
  // Items = (merge task, q head) pairs, dealt round-robin to the warps; lane
  // owns elements [lane*EPL, lane*EPL + EPL) of the item's head.  An item loads
  // all its warp pieces from shared memory at once and combines them against
  // one common maximum, in warp order (deterministic).  A row wholly inside the
  // CTA is normalised and stored (mode 0); a row cut across CTAs leaves its CTA
  // piece in the workspace for planned_xmerge_kernel, next on the stream
  // (mode 1).
  __syncthreads();   // every warp's pieces are in shared memory
  stamp(5);
  const int PS = piece_stride(g, D);   // floats per global piece slot
  const int n_items = (t_end - t_beg) * g;
  // Straight-line, branch-free per item: this phase runs on the layer's critical
  // path and is bound by issue and shared-memory bandwidth (all 8 warps run it
  // together; measured ~1100 -> ~840 SM cycles per item, Llama-70B TP8 17.6 ->
  // 16.8 us per layer, against the divisions, guarded loads and data-dependent
  // branches of a generic version): item it = warp + k W is
  // (task i, head j), advanced incrementally; slots past the task's last piece
  // are not read and weigh nothing (m = -inf, l = o = 0).
  const int qW = W / g, rW = W - qW * g;
  int i = warp / g, j = warp - (warp / g) * g;
  for (int it = warp; it < n_items; it += W) {
    const int4 ta = task_s[2 * i], tb = task_s[2 * i + 1];
    const int wa = ta.z & 0xff, np = ((ta.z >> 8) & 0xff) - wa, wa_slot = (ta.z >> 16) & 1;
    const uint32_t p0 = base + wa * ws.total;                 // warp wa's region
    const uint32_t p0c = p0 + (wa_slot ? ws.ring : ws.piece);  // piece 0: ring slot or piece area
    const uint32_t p1c = p0 + ws.piece;                        // pieces 1..: piece areas of warps wa+u
    const uint32_t off_o = (j * D + lane * EPL) * 4, off_ml = (g * D + 2 * j) * 4;
    float m[kPlannedWarps], l[kPlannedWarps], o[kPlannedWarps][EPL];
#pragma unroll
    for (int u = 0; u < kPlannedWarps; ++u) {   // predicated loads: only the task's pieces (smem bandwidth)
      const uint32_t pc = u == 0 ? p0c : p1c + u * ws.total;
      uint2 ml = make_uint2(0xff800000u, 0u);     // (-inf, 0): an empty slot
      if (u <= np) ml = lds64(pc + off_ml);
      m[u] = __uint_as_float(ml.x);
      l[u] = __uint_as_float(ml.y);
      if constexpr (EPL == 4) {
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (u <= np) v = lds128(pc + off_o);
        o[u][0] = __uint_as_float(v.x);
        o[u][1] = __uint_as_float(v.y);
        o[u][2] = __uint_as_float(v.z);
        o[u][3] = __uint_as_float(v.w);
      } else {
        uint2 v = make_uint2(0u, 0u);
        if (u <= np) v = lds64(pc + off_o);
        o[u][0] = __uint_as_float(v.x);
        o[u][1] = __uint_as_float(v.y);
      }
    }
    float Mb = -1e30f;   // a piece with l > 0 has a finite maximum; empty slots carry -inf
#pragma unroll
    for (int u = 0; u < kPlannedWarps; ++u) Mb = fmaxf(Mb, m[u]);
    float Lr = 0.f, O[EPL];
#pragma unroll
    for (int e = 0; e < EPL; ++e) O[e] = 0.f;
#pragma unroll
    for (int u = 0; u < kPlannedWarps; ++u) {
      const float w = ex2(m[u] - Mb);   // 0 for an empty slot
      Lr = fmaf(l[u], w, Lr);
#pragma unroll
      for (int e = 0; e < EPL; ++e) O[e] = fmaf(o[u][e], w, O[e]);
    }
    if (ta.w == 0) {
      store_row(ta.x, ta.y * g + j, O, rcp_pos(Lr));
    } else {
      float *gp = p.gpiece + static_cast<int64_t>(tb.w) * PS;
      if constexpr (EPL == 4)
        *reinterpret_cast<float4 *>(gp + j * D + lane * EPL) = make_float4(O[0], O[1], O[2], O[3]);
      else
        *reinterpret_cast<float2 *>(gp + j * D + lane * EPL) = make_float2(O[0], O[1]);
      if (lane == 0) *reinterpret_cast<float2 *>(gp + g * D + 2 * j) = make_float2(Mb, Lr);
    }
    i += qW;   // next item of this warp: it + W
    j += rW;
    if (j >= g) {
      j -= g;
      ++i;
    }
  }
  stamp(6);
}

// Cross-CTA merge as a second, stream-ordered kernel:
// one warp per (row cut across CTAs, q head) loads the row's n CTA pieces at once
// and combines them in CTA order.  It needs no atomics or fences -- the decode
// grid has completed -- and its CTAs hold no shared memory, so they co-reside
// with the next layer's decode CTAs, whose pre-wait work (plan, block table,
// early KV tiles) overlaps this kernel.
template <int D>
__global__ void __launch_bounds__(256) planned_xmerge_kernel(const PlannedParams p) {
  constexpr int EPL = D / 32;
  if (p.pdl) asm volatile("griddepcontrol.launch_dependents;");
  const int lane = threadIdx.x & 31;
  const int item = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int g = p.g;
  if (item >= __ldg(p.plan_hdr + offsetof(PlanHeader, n_xrows) / 4) * g) {
    if (p.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
    return;
  }
  const int xr = item / g, j = item - xr * g;
  const int4 x = __ldg(p.xrows + xr);   // plan data: read before the grid wait
  if (p.pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  const int r = x.x, h = x.y, c0 = x.z, n = x.w & 0xffff, flag0 = x.w >> 16;
  const int PS = piece_stride(g, D);
  // the row's CTA pieces in CTA order, 8 loads in flight per batch, branch-free
  // (predicated loads, empty slots weigh nothing), rescaled across batches
  float M = -1e30f, Lr = 0.f, O[EPL];
#pragma unroll
  for (int e = 0; e < EPL; ++e) O[e] = 0.f;
  for (int k0 = 0; k0 < n; k0 += 8) {
    float m[8], l[8], o[8][EPL];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int kk = k0 + u;
      const float *q = p.gpiece + static_cast<int64_t>(kk == 0 ? 2 * c0 + flag0 : 2 * (c0 + kk)) * PS;
      float2 ml = make_float2(-INFINITY, 0.f);
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (kk < n) {
        ml = __ldg(reinterpret_cast<const float2 *>(q + g * D + 2 * j));
        if constexpr (EPL == 4) {
          v = __ldg(reinterpret_cast<const float4 *>(q + j * D + lane * EPL));
        } else {
          const float2 v2 = __ldg(reinterpret_cast<const float2 *>(q + j * D + lane * EPL));
          v.x = v2.x;
          v.y = v2.y;
        }
      }
      m[u] = ml.x;
      l[u] = ml.y;
      o[u][0] = v.x;
      o[u][1] = v.y;
      if constexpr (EPL == 4) {
        o[u][2] = v.z;
        o[u][3] = v.w;
      }
    }
    float Mb = M;
#pragma unroll
    for (int u = 0; u < 8; ++u) Mb = fmaxf(Mb, m[u]);
    const float a = ex2(M - Mb);
    Lr *= a;
#pragma unroll
    for (int e = 0; e < EPL; ++e) O[e] *= a;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float w = ex2(m[u] - Mb);
      Lr = fmaf(l[u], w, Lr);
#pragma unroll
      for (int e = 0; e < EPL; ++e) O[e] = fmaf(o[u][e], w, O[e]);
    }
    M = Mb;
  }
  const float inv = rcp_pos(Lr);
  const int64_t off = static_cast<int64_t>(r) * p.o_ss + static_cast<int64_t>(h * g + j) * p.o_sh + lane * EPL;
  if constexpr (EPL == 4) {
    uint2 w;
    w.x = pack_bf16(O[0] * inv, O[1] * inv);
    w.y = pack_bf16(O[2] * inv, O[3] * inv);
    *reinterpret_cast<uint2 *>(p.out + off) = w;
    peer_put8(p, off, w);
  } else {
    const uint32_t w = pack_bf16(O[0] * inv, O[1] * inv);
    *reinterpret_cast<uint32_t *>(p.out + off) = w;
    peer_put4(p, off, w);
  }
}

}  // namespace planned

int planned_piece_floats(int group, int head_dim) { return planned::piece_stride(group, head_dim); }

int planned_smem_bytes(int head_dim, int group, int slots, int warps) {
  const int gmax = group > 8 ? 16 : 8;
  return 1024 + warps * planned::warp_smem(head_dim, gmax, slots).total;
}

template <int D, bool G16>
static cudaError_t launch_planned_t(const CUtensorMap &tmK, const CUtensorMap &tmV, const PlannedParams &p,
                                   int grid, int warps, int smem, cudaStream_t s) {
  cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void *>(planned::planned_kernel<D, G16>), smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t lc = {};
  cudaLaunchAttribute attr[1];
  lc.gridDim = dim3(grid);
  lc.blockDim = dim3(warps * 32);
  lc.dynamicSmemBytes = smem;
  lc.stream = s;
  if (p.pdl) {
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
  }
  e = cudaLaunchKernelEx(&lc, planned::planned_kernel<D, G16>, tmK, tmV, p);
  if (e != cudaSuccess) return e;
  {   // cross-CTA merge kernel, sized by capacity (graph-safe); items beyond the step's count exit
    cudaLaunchConfig_t lm = {};
    lm.gridDim = dim3((p.xrows_cap * p.g + 7) / 8);
    lm.blockDim = dim3(256);
    lm.stream = s;
    if (p.pdl) {
      lm.attrs = attr;
      lm.numAttrs = 1;
    }
    e = cudaLaunchKernelEx(&lm, planned::planned_xmerge_kernel<D>, p);
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

cudaError_t launch_planned(const CUtensorMap &tmK, const CUtensorMap &tmV, const PlannedParams &p,
                           int head_dim, int grid, int warps, int smem, cudaStream_t s) {
  const bool g16 = p.g > 8;
  if (head_dim == 128)
    return g16 ? launch_planned_t<128, true>(tmK, tmV, p, grid, warps, smem, s)
               : launch_planned_t<128, false>(tmK, tmV, p, grid, warps, smem, s);
  return g16 ? launch_planned_t<64, true>(tmK, tmV, p, grid, warps, smem, s)
             : launch_planned_t<64, false>(tmK, tmV, p, grid, warps, smem, s);
}

}  // namespace bkv
