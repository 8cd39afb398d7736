// decode_attention.cu -- paged decode attention over BROS's bidirectional KV
// cache.
//
// What it computes (reading of SURVEY §8(c) step 5): for request r,
// query head h, kv head h/g:  out = softmax_t(scale * q.K_t) . V_t over the
// request's resident tokens t < L_r, read through the block table and the
// same-shaped direction table.  Attention is a weighted sum over the token
// SET, so this kernel consumes every block in physical slot order; the
// direction only selects which slots of a partly filled block are live
// (forward entry: slots [0, n), reversed entry: slots [bs-n, bs)).  That is
// why the paper's PTX value-vector reversal has no counterpart here.
//
// Design (B200, DESIGN.md §6 "decode attention"):
//  * Persistent grid, one CTA per SM, 8 independent warps per CTA.  Each warp
//    is its own producer: lane 0 streams 16-slot "chunks" (K and V tile of one
//    (block, kv head), 2*d*32 bytes) through a private 2-deep ring of
//    128B-swizzled shared-memory slots -- ONE 5-D TMA box per chunk when the
//    pool allows a combined K|V view, else one per tile -- with mbarrier
//    completion; the consumer moves the tile to registers and refills the
//    slot before doing the math.
//  * Work units = (request, kv head, split of <= P blocks), pulled from a
//    global atomic counter (first unit static), enumerated longest-first by a
//    4-bucket split plan computed in-kernel from seq_lens (entry counts for
//    general maps); small problems get a chain-balanced P, or -- when warp
//    ranges would hold >= 12 blocks -- the stream-K plan: the flattened
//    (request, kv head, block) sequence cut into equal contiguous ranges, one
//    per warp, whose row segments are the units (rows cut across ranges leave
//    per-range partial slots).  The issuer decodes the next unit one unit
//    ahead (block-table window loads, q L2 prefetch).
//  * PDL: both kernels trigger their dependents at entry; the plan prologue
//    reads only seq_lens (and entry counts) before griddepcontrol.wait.
//  * Tensor cores for every group size (the CUDA-core FFMA2 MHA variant is a
//    dev switch, BKV_MHA_CUDA_CORES=1): tokens on the MMA M dimension,
//    S^T = K.Q^T and O^T += V^T.P^T with bf16 mma.sync m16n8k16 (K via
//    ldmatrix, V via ldmatrix.trans, P^T re-laid through 256 B of smem).
//  * A unit's output is written directly when the request has one split;
//    otherwise fp32 (m, l, o) partials go to the workspace and merge_kernel,
//    stream-ordered after this kernel, combines them in split order (an
//    in-kernel last-arriver merge exists behind BKV_FUSED_MERGE=1).
//  * Fused decode step (bkv_decode_step): the chunk that
//    holds a unit's new token t = L-1 also bulk-loads the token's K/V rows
//    (from k_new/v_new) into a per-slot patch area on the same mbarrier; the
//    consumer writes them into the tile's slot row (128B swizzle) and bulk-
//    stores them into the pool -- the append costs no extra launch and no
//    ordering stall.
//  * NaN hygiene (reading Q10): dead slots are never combined arithmetically:
//    their scores are selected to -inf and their V rows are zeroed in shared
//    memory before P.V.
#include <math.h>

#include "bkv_internal.h"
#include "bkv_ptx.cuh"

namespace bkv {

// Dev-only timeline / cycle tracing (scripts/trace_run.py): compiled in only
// when libbkv is built with BKV_BUILD_TRACE=1 (-DBKV_DEV_TRACE), so the product
// kernel carries neither the code nor the registers.
#ifdef BKV_DEV_TRACE
constexpr bool kDevTrace = true;
#else
constexpr bool kDevTrace = false;
#endif

// F_NEW (fused decode step): the chunk holds this step's new token; its slot
// in the block sits in flags bits 8..15 and the physical block in SlotMeta::aux.
enum : int { F_FIRST = 1, F_LAST = 2, F_NOKV = 4, F_NOQ = 8, F_NEW = 16 };

struct SlotMeta {
  int u, r, h, nsplit;
  int lo, hi, flags, aux;
};

constexpr int kBuckets = 4;
constexpr int kFastSplits = 8;   // merge: rows with <= this many splits preload every partial
constexpr int kStreamKMinRange = 12;   // stream-K plan only when warp ranges are at least this long

struct Plan {
  int P;                  // target blocks per split
  int base[kBuckets + 1]; // split-slot offset of each size bucket (largest first)
  int U;                  // units = base[kBuckets] * H (stream-K: 2 partial slots per warp)
  int streamk;            // 1: stream-K plan -- P = blocks per warp range, Pre[0] = prefix of nb
};

template <int D>
struct Geo {
  static constexpr int HALVES = D / 64;        // 64-element (128 B) swizzle atoms per row
  static constexpr int HALF_BYTES = 16 * 128;  // 16 slots x 128 B
  static constexpr int KV_BYTES = HALVES * HALF_BYTES;
  static constexpr int SLOT_BYTES = 2 * KV_BYTES;
};

// 128B swizzle: 16-byte piece c of row `row` sits at piece c ^ (row & 7).
__device__ __forceinline__ uint32_t swz(int row, int c) {
  return static_cast<uint32_t>(row * 128 + ((c ^ (row & 7)) << 4));
}

__device__ __forceinline__ int nblocks_of(int L, int bs) { return L > 0 ? (L + bs - 1) / bs : 0; }

// Largest index i in [0, n] with a[i] <= x (a non-decreasing, a[0] = 0 <= x).
__device__ __forceinline__ int search_le(const int *a, int n, int x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (a[mid] <= x)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

// Split plan, computed identically by every CTA from
// seq_lens (no host round trip).  P = ceil(sum_r nb_r * H / target) blocks
// when that is >= min_split, else the small-problem rule below; request r is cut into n_r = ceil(nb_r / P) near-equal
// splits of s_r <= P blocks.  Requests are grouped into 4 buckets by split
// size (largest first) and units are enumerated bucket by bucket, so the
// dynamically scheduled work list runs roughly longest-first and the tail is
// made of small units.  Pre[k][r] = exclusive prefix of n_r over bucket k.
__device__ __forceinline__ int bucket_of(int s, int P) {
  // s in (3P/4, P] -> 0, (P/2, 3P/4] -> 1, (P/4, P/2] -> 2, [0, P/4] -> 3
  return 4 * s > 3 * P ? 0 : (2 * s > P ? 1 : (4 * s > P ? 2 : 3));
}

// Entries (blocks) of request r: ceil(L/bs) for a dense map, num_entries[r]
// for a general one.
__device__ __forceinline__ int entries_of(const DecodeParams &p, int r, int L) {
  return p.fills ? __ldg(p.nent + r) : nblocks_of(L, p.bs);
}

// ceil(a / b), 0 <= a, 1 <= b: a 32-bit unsigned division when both fit (the
// usual case -- the 64-bit one is a software routine of several hundred cycles
// on the prologue's critical path)
__device__ __forceinline__ long long cdiv_ll(long long a, long long b) {
  if (((static_cast<unsigned long long>(a) | static_cast<unsigned long long>(b)) >> 32) == 0) {
    const unsigned ua = static_cast<unsigned>(a), ub = static_cast<unsigned>(b);
    const unsigned q = ua / ub;
    return q + (q * ub != ua ? 1 : 0);
  }
  return (a + b - 1) / b;
}

// splits of a request with nb entries and its size bucket, packed (n << 2 | bucket)
__device__ __forceinline__ int split_code(int nb, int P) {
  const unsigned n = nb > 0 ? (static_cast<unsigned>(nb) + P - 1) / static_cast<unsigned>(P) : 1u;
  const unsigned sz = (static_cast<unsigned>(nb) + n - 1) / n;
  return static_cast<int>(n << 2) | bucket_of(static_cast<int>(sz), P);
}

__device__ void compute_plan(const DecodeParams &p, int *Pre, int *Lsm, int *NBsm, Plan *plan,
                             long long *pc = nullptr) {   // pc: dev trace clocks
  __shared__ long long red_ll[32];
  __shared__ int4 red4[32];
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5,
            nw = nt >> 5;
  const int B = p.B;
  long long local = 0;
  for (int r = tid; r < B; r += nt) {
    const int L = __ldg(p.seq_lens + r);
    const int nb = entries_of(p, r, L);
    Lsm[r] = L;
    NBsm[r] = nb;
    local += nb;
  }
  if (kDevTrace && pc) pc[0] = clock64();
#pragma unroll
  for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if (lane == 0) red_ll[warp] = local;
  __syncthreads();
  if (kDevTrace && pc) pc[1] = clock64();
  long long T = 0;
  for (int w = 0; w < nw; ++w) T += red_ll[w];
  const long long target = max(1, p.target_units);
  long long Pll = cdiv_ll(T * p.H, target);
  if (Pll < p.min_split) {
    // Small problem (fewer than ~3 min_split-block units per warp): the step is
    // bounded by the longest per-warp chain, not by bandwidth.  Units number at
    // most TH/P + BH (each (r, h) rounds up once), so P_k = ceil(TH / (kW - BH))
    // gives every warp at most k units; pick k in {1, 2, 3} minimising the
    // chain k * (P_k + 2) (a unit's q load + output cost about two chunks).
    const long long TH = T * p.H, BH = static_cast<long long>(p.B) * p.H, W = p.total_warps;
    long long best = -1, bestP = p.min_split;
    for (int k = 1; k <= 3; ++k) {
      const long long room = k * W - BH;
      if (room <= 0) continue;
      const long long Pk = max(1ll, cdiv_ll(TH, room));
      if (Pk > p.min_split) continue;
      const long long chain = k * (Pk + 2);
      if (best < 0 || chain < best) {
        best = chain;
        bestP = Pk;
      }
    }
    Pll = p.small_plan ? bestP : p.min_split;
    // stream-K when a warp's range holds >= kStreamKMinRange blocks (measured:
    // Llama-70B TP2 65.3 -> 60.5 us, TP4 37.7 -> 35.1, OPT-13B TP4 39.0 -> 37.5; with
    // ~8-block ranges (TP8 shards) the extra segments cost more than the balance gains)
    if (p.streamk == 1 && TH >= static_cast<long long>(kStreamKMinRange) * W) Pll = -1;
  }
  if (p.streamk == 2) Pll = -1;   // dev: stream-K for every problem size
  const bool sk = Pll < 0;
  // stream-K (small problems): the flattened (request, kv head, block)
  // sequence is cut into equal ranges of P blocks, one per warp; the scans below then
  // give Pre[0][r] = sum of nb over requests before r (all "splits" in bucket 0)
  const int P = sk ? static_cast<int>(max(1ll, cdiv_ll(T * p.H, static_cast<long long>(p.total_warps))))
                   : static_cast<int>(Pll);
  if (kDevTrace && pc) pc[2] = clock64();
  // per-thread contiguous ranges -> 4-bucket exclusive scans of n_r
  const int per = (B + nt - 1) / nt;
  const int r0 = min(B, tid * per), r1 = min(B, r0 + per);
  int4 cnt = make_int4(0, 0, 0, 0);
  int *code = Pre + 3 * (B + 1);   // split codes, parked in Pre[3][r] until this thread overwrites them
  for (int r = r0; r < r1; ++r) {
    const int c = sk ? (NBsm[r] << 2) : split_code(NBsm[r], P);
    code[r] = c;
    const int n = c >> 2, bk = c & 3;
    cnt.x += bk == 0 ? n : 0;
    cnt.y += bk == 1 ? n : 0;
    cnt.z += bk == 2 ? n : 0;
    cnt.w += bk == 3 ? n : 0;
  }
  int4 inc = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int x = __shfl_up_sync(0xffffffffu, inc.x, o), y = __shfl_up_sync(0xffffffffu, inc.y, o);
    const int z = __shfl_up_sync(0xffffffffu, inc.z, o), w = __shfl_up_sync(0xffffffffu, inc.w, o);
    if (lane >= o) {
      inc.x += x;
      inc.y += y;
      inc.z += z;
      inc.w += w;
    }
  }
  if (lane == 31) red4[warp] = inc;
  __syncthreads();
  if (kDevTrace && pc) pc[3] = clock64();
  int4 e = make_int4(inc.x - cnt.x, inc.y - cnt.y, inc.z - cnt.z, inc.w - cnt.w);
  for (int w = 0; w < warp; ++w) {
    e.x += red4[w].x;
    e.y += red4[w].y;
    e.z += red4[w].z;
    e.w += red4[w].w;
  }
  for (int r = r0; r < r1; ++r) {
    const int c = code[r];
    const int n = c >> 2, bk = c & 3;
    Pre[0 * (B + 1) + r] = e.x;
    Pre[1 * (B + 1) + r] = e.y;
    Pre[2 * (B + 1) + r] = e.z;
    Pre[3 * (B + 1) + r] = e.w;
    e.x += bk == 0 ? n : 0;
    e.y += bk == 1 ? n : 0;
    e.z += bk == 2 ? n : 0;
    e.w += bk == 3 ? n : 0;
  }
  if (tid == nt - 1) {
    int4 tot = make_int4(0, 0, 0, 0);
    for (int w = 0; w < nw; ++w) {
      tot.x += red4[w].x;
      tot.y += red4[w].y;
      tot.z += red4[w].z;
      tot.w += red4[w].w;
    }
    Pre[0 * (B + 1) + B] = tot.x;
    Pre[1 * (B + 1) + B] = tot.y;
    Pre[2 * (B + 1) + B] = tot.z;
    Pre[3 * (B + 1) + B] = tot.w;
    plan->base[0] = 0;
    plan->base[1] = tot.x;
    plan->base[2] = tot.x + tot.y;
    plan->base[3] = tot.x + tot.y + tot.z;
    const int acc = tot.x + tot.y + tot.z + tot.w;
    plan->base[kBuckets] = acc;
    plan->P = P;
    plan->U = sk ? 2 * p.total_warps : acc * p.H;
    plan->streamk = sk ? 1 : 0;
  }
  __syncthreads();
}

// Merge of the split partials of one (request r, kv head h, q head `head` of
// the group) row, in split order: M = max m_s, L = sum l_s 2^(m_s - M),
// O = sum o_s 2^(m_s - M) / L.  Lanes take 32 splits at a
// time, weights are broadcast by shuffle, each lane owns EPL output elements.
// COHERENT: the partials were written by other SMs during THIS kernel (fused
// last-arriver merge) -> L2 loads (ld.global.cg), else read-only cached loads.
template <int D, bool COHERENT>
__device__ __forceinline__ void merge_row(const DecodeParams &p, int u0, int ns, int r, int h, int head,
                                          int lane, int u_first, int ustride) {
  // split s of the row lives in unit slot (s == 0 ? u_first : u0 + s * ustride)
  auto unit_of = [&](int sidx) { return sidx == 0 ? u_first : u0 + sidx * ustride; };
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int EPL = D / 32;
  const int g = p.g;
  float Mrun = -INFINITY, Lrun = 0.f, acc[EPL];
#pragma unroll
  for (int q = 0; q < EPL; ++q) acc[q] = 0.f;
  if (!COHERENT && ns <= kFastSplits) {   // (the fused in-kernel merge keeps the register-light loop)
    // Few splits (the common case): every partial load -- all (m, l) pairs and
    // all o slices -- is issued before any of them is used, so the row costs
    // one memory round trip instead of two.
    float ov[kFastSplits][EPL];
#pragma unroll
    for (int t = 0; t < kFastSplits; ++t) {
      if (t < ns) {
        const float *po = p.part_o + (static_cast<int64_t>(unit_of(t)) * g + head) * D + lane * EPL;
        if constexpr (EPL == 4) {
          const float4 v = COHERENT ? __ldcg(reinterpret_cast<const float4 *>(po)) : __ldg(reinterpret_cast<const float4 *>(po));
          ov[t][0] = v.x;
          ov[t][1] = v.y;
          ov[t][2] = v.z;
          ov[t][3] = v.w;
        } else {
          const float2 v = COHERENT ? __ldcg(reinterpret_cast<const float2 *>(po)) : __ldg(reinterpret_cast<const float2 *>(po));
          ov[t][0] = v.x;
          ov[t][1] = v.y;
        }
      }
    }
    float wj = -INFINITY, lj = 0.f;
    if (lane < ns) {
      const float2 *src = reinterpret_cast<const float2 *>(p.part_ml + (static_cast<int64_t>(unit_of(lane)) * g + head) * 2);
      const float2 v = COHERENT ? __ldcg(src) : __ldg(src);
      wj = v.x;
      lj = v.y;
    }
    float mg = wj;
#pragma unroll
    for (int o = 16; o; o >>= 1) mg = fmaxf(mg, __shfl_xor_sync(FULL, mg, o));
    const float w = lane < ns ? ex2(wj - mg) : 0.f;
    float ls = lj * w;
#pragma unroll
    for (int o = 16; o; o >>= 1) ls += __shfl_xor_sync(FULL, ls, o);
    Lrun = ls;
#pragma unroll
    for (int t = 0; t < kFastSplits; ++t) {
      const float wt = __shfl_sync(FULL, w, t);
      if (t < ns) {
#pragma unroll
        for (int q = 0; q < EPL; ++q) acc[q] = fmaf(wt, ov[t][q], acc[q]);
      }
    }
  }
  for (int s0 = 0; (COHERENT || ns > kFastSplits) && s0 < ns; s0 += 32) {
    const int sl = s0 + lane;
    const bool ok = sl < ns;
    const int us = unit_of(sl);
    float wj = -INFINITY, lj = 0.f;
    if (ok) {
      const float2 *src = reinterpret_cast<const float2 *>(p.part_ml + (static_cast<int64_t>(us) * g + head) * 2);
      const float2 v = COHERENT ? __ldcg(src) : __ldg(src);
      wj = v.x;
      lj = v.y;
    }
    float mg = wj;
#pragma unroll
    for (int o = 16; o; o >>= 1) mg = fmaxf(mg, __shfl_xor_sync(FULL, mg, o));
    const float Mn = fmaxf(Mrun, mg);
    const float a = ex2(Mrun - Mn);
    const float w = ok ? ex2(wj - Mn) : 0.f;
    float ls = lj * w;
#pragma unroll
    for (int o = 16; o; o >>= 1) ls += __shfl_xor_sync(FULL, ls, o);
    Lrun = Lrun * a + ls;
#pragma unroll
    for (int q = 0; q < EPL; ++q) acc[q] *= a;
    Mrun = Mn;
    const int cnt = min(32, ns - s0);
#pragma unroll 4
    for (int t = 0; t < cnt; ++t) {
      const int ut = __shfl_sync(FULL, us, t);
      const float wt = __shfl_sync(FULL, w, t);
      const float *po = p.part_o + (static_cast<int64_t>(ut) * g + head) * D + lane * EPL;
      if constexpr (EPL == 4) {
        const float4 v = COHERENT ? __ldcg(reinterpret_cast<const float4 *>(po)) : __ldg(reinterpret_cast<const float4 *>(po));
        acc[0] = fmaf(wt, v.x, acc[0]);
        acc[1] = fmaf(wt, v.y, acc[1]);
        acc[2] = fmaf(wt, v.z, acc[2]);
        acc[3] = fmaf(wt, v.w, acc[3]);
      } else {
        const float2 v = COHERENT ? __ldcg(reinterpret_cast<const float2 *>(po)) : __ldg(reinterpret_cast<const float2 *>(po));
        acc[0] = fmaf(wt, v.x, acc[0]);
        acc[1] = fmaf(wt, v.y, acc[1]);
      }
    }
  }
  const float inv = Lrun > 0.f ? 1.f / Lrun : 0.f;
  const int64_t off = static_cast<int64_t>(r) * p.o_ss + static_cast<int64_t>(h * g + head) * p.o_sh + lane * EPL;
  if constexpr (EPL == 4) {
    uint2 w;
    w.x = pack_bf16(acc[0] * inv, acc[1] * inv);
    w.y = pack_bf16(acc[2] * inv, acc[3] * inv);
    *reinterpret_cast<uint2 *>(p.out + off) = w;
    peer_put8(p, off, w);
  } else {
    const uint32_t w = pack_bf16(acc[0] * inv, acc[1] * inv);
    *reinterpret_cast<uint32_t *>(p.out + off) = w;
    peer_put4(p, off, w);
  }
}

// Merge of ALL g rows of (r, h) by one warp (the fused last-arriver path, g <= 8):
// the (m, l) of every (split, row) pair are loaded at once into the warp's
// shared scratch, lanes < g turn them into normalised weights
// w = 2^(m - M) / L, then each lane accumulates its EPL output elements of
// every row with all partial loads of a split issued together (no per-row
// dependent chain).  Same result as merge_row up to fp32 rounding order.
template <int D>
__device__ __forceinline__ void merge_group(const DecodeParams &p, int u0, int ns, int r, int h, int lane,
                                            uint32_t scr) {
  constexpr int EPL = D / 32;
  const int H = p.H, g = p.g;
  for (int idx = lane; idx < ns * g; idx += 32) {
    const int sp = idx / g, j = idx - sp * g;
    const float2 v = __ldcg(reinterpret_cast<const float2 *>(
        p.part_ml + (static_cast<int64_t>(u0 + sp * H) * g + j) * 2));
    st_shared_v2f(scr + idx * 8, v.x, v.y);
  }
  __syncwarp();
  if (lane < g) {
    float M = -INFINITY;
    for (int sp = 0; sp < ns; ++sp) M = fmaxf(M, __uint_as_float(lds32(scr + (sp * g + lane) * 8)));
    float Ls = 0.f;
    for (int sp = 0; sp < ns; ++sp) {
      const uint32_t a = scr + (sp * g + lane) * 8;
      Ls += __uint_as_float(lds32(a + 4)) * ex2(__uint_as_float(lds32(a)) - M);
    }
    const float inv = Ls > 0.f ? 1.f / Ls : 0.f;
    for (int sp = 0; sp < ns; ++sp) {
      const uint32_t a = scr + (sp * g + lane) * 8;
      st_shared_f32(a, ex2(__uint_as_float(lds32(a)) - M) * inv);   // weight replaces m
    }
  }
  __syncwarp();
  float acc[8][EPL];
#pragma unroll
  for (int j = 0; j < 8; ++j)
#pragma unroll
    for (int q = 0; q < EPL; ++q) acc[j][q] = 0.f;
  for (int sp = 0; sp < ns; ++sp) {
    const float *po = p.part_o + static_cast<int64_t>(u0 + sp * H) * g * D + lane * EPL;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (j >= g) break;
      const float w = __uint_as_float(lds32(scr + (sp * g + j) * 8));
      if constexpr (EPL == 4) {
        const float4 v = __ldcg(reinterpret_cast<const float4 *>(po + j * D));
        acc[j][0] = fmaf(w, v.x, acc[j][0]);
        acc[j][1] = fmaf(w, v.y, acc[j][1]);
        acc[j][2] = fmaf(w, v.z, acc[j][2]);
        acc[j][3] = fmaf(w, v.w, acc[j][3]);
      } else {
        const float2 v = __ldcg(reinterpret_cast<const float2 *>(po + j * D));
        acc[j][0] = fmaf(w, v.x, acc[j][0]);
        acc[j][1] = fmaf(w, v.y, acc[j][1]);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (j >= g) break;
    uint16_t *o = p.out + static_cast<int64_t>(r) * p.o_ss + static_cast<int64_t>(h * g + j) * p.o_sh + lane * EPL;
    if constexpr (EPL == 4) {
      uint2 w2;
      w2.x = pack_bf16(acc[j][0], acc[j][1]);
      w2.y = pack_bf16(acc[j][2], acc[j][3]);
      *reinterpret_cast<uint2 *>(o) = w2;
    } else {
      *reinterpret_cast<uint32_t *>(o) = pack_bf16(acc[j][0], acc[j][1]);
    }
  }
  __syncwarp();
}

// KIND 0: MHA on CUDA cores; 1: MMA with g <= 8; 2: MMA with 8 < g <= 16.
// GQA runs 8 warps (measured best) and gets the 255-register budget of a
// 256-thread CTA -- at 384 threads the MMA kernels spill (ptxas -v).
template <int D, int KIND>
__global__ void __launch_bounds__(KIND == 0 ? 384 : 256, 1)
    decode_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                  const DecodeParams p) {
  using G = Geo<D>;
  constexpr bool MMA = KIND != 0;
  constexpr bool G16 = KIND == 2;
  constexpr unsigned FULL = 0xffffffffu;

  extern __shared__ uint8_t smem_raw[];
  __shared__ Plan plan;
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t *gbase = smem_raw + (base - raw);
  const int W = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int S = p.slots;
  const uint32_t slots_base = base;
  uint8_t *meta_g = gbase + W * S * G::SLOT_BYTES;
  SlotMeta *metas = reinterpret_cast<SlotMeta *>(meta_g) + warp * S;
  uint64_t *bars_g = reinterpret_cast<uint64_t *>(meta_g + W * S * sizeof(SlotMeta));
  uint8_t *scratch_g = reinterpret_cast<uint8_t *>(bars_g + W * S);   // W x 1 KiB
  const uint32_t my_scr = smem_u32(scratch_g + warp * 1024);
  uint8_t *patch_g = scratch_g + W * 1024;                    // W x S x 512 B: new K|V rows
  const uint32_t my_patch = smem_u32(patch_g + warp * S * 512);
  int *Pre = reinterpret_cast<int *>(patch_g + W * S * 512);  // [kBuckets][B + 1]
  int *Lsm = Pre + kBuckets * (p.B + 1);                      // seq_lens cache [B]
  int *NBsm = Lsm + ((p.B + 3) & ~3);                         // entries per request [B]

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmK);
    prefetch_tmap(&tmV);
  }
  // dev-only event trace: (globaltimer ns << 8 | kind), unit id in a second word
  int trace_n = 0;
  auto trace = [&](int kind, int u) {
    if (kDevTrace && p.trace && lane == 0 && trace_n < p.trace_cap) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      unsigned long long *e = p.trace + (static_cast<int64_t>(blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * p.trace_cap + trace_n) * 2;
      e[0] = (t << 8) | kind;
      e[1] = static_cast<unsigned long long>(u);
      ++trace_n;
    }
  };
  trace(0, -1);
  // PDL: let the stream's next kernel (the merge) be scheduled onto SMs as
  // this grid's CTAs exit; it still waits for this whole grid to complete
  if (p.pdl && !(p.debug_flags & 32)) asm volatile("griddepcontrol.launch_dependents;");
  if (p.debug_flags & 16) return;   // dev: launch cost only
  long long pc[6];
  pc[5] = kDevTrace ? clock64() : 0;
  compute_plan(p, Pre, Lsm, NBsm, &plan, kDevTrace ? pc : nullptr);
  if (kDevTrace) {
    pc[4] = clock64();
    for (int k = 0; k < 5; ++k) trace(16 + k, static_cast<int>(pc[k] - pc[5]));
  }
  // PDL: everything above read only seq_lens; wait for the preceding kernel
  // (it may have written the pool / q) before touching anything else.
  if (p.pdl && !p.pdl_nowait) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (blockIdx.x == 0) {   // publish the split plan for the merge kernel
    if (threadIdx.x == 0) {
      p.plan_out[0] = plan.P;
      for (int k = 0; k <= kBuckets; ++k) p.plan_out[1 + k] = plan.base[k];
      p.plan_out[6] = plan.U;
      p.plan_out[7] = plan.streamk;
    }
    // per request: (first split slot, split count) -> the merge kernel needs one load per row
    // (stream-K: (blocks before the request, its blocks))
    for (int r = threadIdx.x; r < p.B; r += blockDim.x) {
      if (plan.streamk) {
        reinterpret_cast<int2 *>(p.plan_out + 16)[r] = make_int2(Pre[r], NBsm[r]);
        continue;
      }
      const int c = split_code(NBsm[r], plan.P), k = c & 3;
      reinterpret_cast<int2 *>(p.plan_out + 16)[r] = make_int2(plan.base[k] + Pre[k * (p.B + 1) + r], c >> 2);
    }
  }
  trace(1, -1);
  if (p.debug_flags & 8) return;    // dev: launch + plan prologue only
  const int P = plan.P, U = plan.U;

  const uint32_t my_slots = slots_base + warp * S * G::SLOT_BYTES;
  const uint32_t my_bars = smem_u32(bars_g + warp * S);
  if (lane == 0) {
    for (int i = 0; i < S; ++i) mbar_init(my_bars + 8 * i, 1);
    fence_mbar_init();
  }
  __syncwarp();
  const uint64_t pol = policy_evict_first();
  const int g = p.g, H = p.H, bs = p.bs;
  const int chunks_per_block = bs >> 4;

  // ------------------------------------------------------------ issuer state
  // First unit static (no atomic storm at launch), later ones pulled from a
  // global counter.  The issuer
  // decodes the NEXT unit and starts its block-table loads when it enters the
  // current one, so unit boundaries do not stall on global memory.
  // first units interleave across SMs (warp-major), so small problems spread over the whole chip
  int u_pref = (p.debug_flags & 4) ? static_cast<int>(blockIdx.x) * W + warp
                                    : warp * static_cast<int>(gridDim.x) + static_cast<int>(blockIdx.x);
  auto pull_unit = [&]() -> int {
    const int u = __shfl_sync(FULL, u_pref, 0);
    if (u < U && lane == 0) u_pref = p.total_warps + atomicAdd(p.sched, 1);  // used one unit later
    return u;
  };
  struct UnitInfo {
    int u, r, h, L, nb, n, e0, e1;
  };
  auto decode_unit = [&](int u) -> UnitInfo {
    UnitInfo x;
    x.u = u;
    if (u >= U) return x;
    x.h = u % H;
    const int qq = u / H;
    int k = 0;
    while (k < kBuckets - 1 && qq >= plan.base[k + 1]) ++k;
    const int j = qq - plan.base[k];
    const int *pk = Pre + k * (p.B + 1);
    x.r = search_le(pk, p.B, j);
    x.L = Lsm[x.r];
    const int nb = NBsm[x.r];
    x.nb = nb;
    x.n = nb > 0 ? (nb + P - 1) / P : 1;
    const int sidx = j - pk[x.r];
    x.e0 = static_cast<int>(static_cast<long long>(sidx) * nb / x.n);
    x.e1 = static_cast<int>(static_cast<long long>(sidx + 1) * nb / x.n);
    return x;
  };
  // window of 32 block-table/direction(/fill) entries starting at block wb (lane i: entry wb + i)
  auto load_window = [&](const UnitInfo &x, int wb, int &btv, int &dirv, int &filv) {
    const int ew = wb + lane;
    btv = 0;
    dirv = 0;
    filv = 0;
    if (x.u < U && ew < x.e1) {
      btv = __ldg(p.bt + static_cast<int64_t>(x.r) * p.bt_stride + ew);
      dirv = __ldg(p.dirs + static_cast<int64_t>(x.r) * p.dir_rs + static_cast<int64_t>(ew) * p.dir_cs);
      if (p.fills) filv = __ldg(p.fills + static_cast<int64_t>(x.r) * p.fill_rs + ew);
    }
  };
  // stream-K plan: this warp's range of the flattened (request, kv head, block)
  // sequence, cut into segments at row boundaries; each segment is a unit
  const int gw = u_pref;   // the warp's static first unit = its range index
  int sk_beg = 0, sk_pos = 0, sk_end = 0;
  if (plan.streamk) {
    const int N = Pre[p.B] * H;   // total blocks x kv heads (Pre[0][B])
    sk_beg = min(N, gw * P);
    sk_pos = sk_beg;
    sk_end = min(N, sk_beg + P);
  }
  auto next_unit = [&]() -> UnitInfo {
    if (!plan.streamk) return decode_unit(pull_unit());
    UnitInfo x;
    x.u = U;
    if (sk_pos >= sk_end) return x;
    const int a = sk_pos;
    x.r = search_le(Pre, p.B, a / H);   // largest r with H * Pre[0][r] <= a (so nb_r > 0)
    x.nb = NBsm[x.r];
    x.L = Lsm[x.r];
    const int off = a - H * Pre[x.r];
    x.h = off / x.nb;
    x.e0 = off - x.h * x.nb;
    x.e1 = min(x.nb, x.e0 + (sk_end - a));
    x.n = (x.e0 == 0 && x.e1 == x.nb) ? 1 : 2;   // whole row: direct output, else a partial
    x.u = 2 * gw + (a == sk_beg ? 0 : 1);        // slot: the range's first / last segment
    sk_pos = a + (x.e1 - x.e0);
    return x;
  };
  UnitInfo cur{}, nxt = next_unit();
  int nx_bt = 0, nx_dir = 0, nx_fil = 0;
  load_window(nxt, nxt.e0, nx_bt, nx_dir, nx_fil);
  bool is_active = false, is_done = false, is_first = false;
  int is_ci = 0, is_nc = 0, is_wb = 0, bt_w = 0, dir_w = 0, fil_w = 0;

  // Produce the next chunk of this warp's work stream (warp-collective).
  // Chunk ci of a unit = 16 slots (sub-chunk ci % cpb) of block e0 + ci / cpb;
  auto next_chunk = [&](SlotMeta &m, int &blk, int &csub) -> bool {
    if (!is_active) {
      if (is_done) return false;
      if (nxt.u >= U) {
        is_done = true;
        return false;
      }
      cur = nxt;
      bt_w = nx_bt;
      dir_w = nx_dir;
      fil_w = nx_fil;
      is_wb = cur.e0;
      nxt = next_unit();                                  // look one unit ahead ...
      load_window(nxt, nxt.e0, nx_bt, nx_dir, nx_fil);    // ... its loads overlap this unit
      if (lane < g) {   // the unit's q rows: pull into L2 now, the consumer loads them later
        const uint16_t *qrow = p.q + static_cast<int64_t>(cur.r) * p.q_ss +
                               static_cast<int64_t>(cur.h * g + lane) * p.q_sh;
        asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(qrow));
        if (D == 128) asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(qrow + 64));
      }
      is_ci = 0;
      is_nc = (cur.e1 - cur.e0) * chunks_per_block;
      is_first = true;
      trace(2, cur.u);
      if (is_ci >= is_nc) {  // no chunk for this warp (or empty context, Q8): flag-only slot
        m = SlotMeta{cur.u, cur.r, cur.h, cur.n, 0, 0, F_FIRST | F_LAST | F_NOKV | F_NOQ, 0};
        blk = 0;
        csub = 0;
        return true;
      }
      is_active = true;
    }
    const int e = cur.e0 + (chunks_per_block == 1 ? is_ci : (is_ci >> 1));
    const int c = chunks_per_block == 1 ? 0 : (is_ci & 1);
    if (e - is_wb >= 32) {  // long unit: refill the window (rare)
      is_wb = e;
      load_window(cur, e, bt_w, dir_w, fil_w);
    }
    const int idx = e - is_wb;
    const int b = __shfl_sync(FULL, bt_w, idx);
    const int dr = __shfl_sync(FULL, dir_w, idx);
    const int fl = __shfl_sync(FULL, fil_w, idx);
    // live tokens in this block: dense map -> all but the last entry full;
    // general map (f3) -> the entry's fill count
    const int ne = p.fills ? fl : min(bs, cur.L - e * bs);
    const int lo_s = dr ? bs - ne : 0;               // RT from the left,
    const int hi_s = dr ? bs : ne;                   //        BE from the right
    const int lo = max(lo_s - c * 16, 0), hi = min(hi_s - c * 16, 16);
    int flags = (is_first ? F_FIRST : 0) | (lo >= hi ? F_NOKV : 0);
    if (p.k_new != nullptr && e == cur.nb - 1) {
      // fused decode step: token t = L-1 of (r, h) is the
      // last token of the last entry, in its direction's slot; this
      // warp alone owns it.
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
    }
    m = SlotMeta{cur.u, cur.r, cur.h, cur.n, lo, hi, flags, b};
    return true;
  };

  auto issue = [&](int i, const SlotMeta &m, int blk, int csub) {
    if (lane == 0) {
      reinterpret_cast<int4 *>(metas + i)[0] = make_int4(m.u, m.r, m.h, m.nsplit);
      reinterpret_cast<int4 *>(metas + i)[1] = make_int4(m.lo, m.hi, m.flags, m.aux);
      const uint32_t bar = my_bars + 8 * i;
      const bool kv = !(m.flags & F_NOKV);
      const bool nw = m.flags & F_NEW;
      const uint32_t bytes = (kv ? G::SLOT_BYTES : 0) + (nw ? 4 * D : 0);
      mbar_arrive_expect_tx(bar, bytes);
      if (nw) {   // the new K and V rows ride on the same barrier into the slot's patch area
        bulk_wait_read_all();   // (the previous bulk store out of this area has read it)
        const int64_t row = (static_cast<int64_t>(m.r) * H + m.h) * D;
        bulk_load(my_patch + i * 512, p.k_new + row, 2 * D, bar);
        bulk_load(my_patch + i * 512 + 2 * D, p.v_new + row, 2 * D, bar);
      }
      if (kv) {
        // one 5-D box = the whole 16-slot x d tile, laid out [half][slot][128 B] swizzled
        const uint32_t dk = my_slots + i * G::SLOT_BYTES, dv = dk + G::KV_BYTES;
        if (p.kv_mode) {   // one box = K and V tiles of (block, head): [kv][half][slot][128 B]
          tma_load_5d(dk, &tmK, 0, csub * 16, 0, 0, blk * H + m.h, bar, pol);
        } else {
          tma_load_5d(dk, &tmK, 0, csub * 16, 0, m.h, blk, bar, pol);
          tma_load_5d(dv, &tmV, 0, csub * 16, 0, m.h, blk, bar, pol);
        }
      }
    }
  };

  // --------------------------------------------------------- consumer state
  constexpr int NCH = D / 16;       // MHA: 16-byte K pieces per lane (lane = token x half of d)
  constexpr int EPL = D / 32;       // output elements per lane (MHA P.V, merge)
  constexpr int NT = G16 ? 2 : 1;   // MMA: 8-head n-tiles
  constexpr int MT = D / 16;        // MMA: 16-element d tiles (= k-steps of Q.K^T)
  float2 o2[MMA ? 1 : EPL / 2];                  // MHA output accumulator (q lives in scratch)
  uint32_t qb[MMA ? MT : 1][NT][2];              // MMA: Q^T B-fragments
  float oacc[MMA ? MT : 1][NT][4];               // MMA: O^T accumulators [d tile][head tile]
  float mrun[NT][2], lrun[NT][2];                // MHA uses [0][0]

  // q of the unit: global loads (the issuer pulled the rows into L2 when it
  // started the unit, several chunks ago)
  auto begin_unit = [&](const SlotMeta &m) {
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      mrun[n][0] = mrun[n][1] = -INFINITY;
      lrun[n][0] = lrun[n][1] = 0.f;
    }
    const bool noq = m.flags & F_NOQ;
    const uint16_t *qg = p.q + static_cast<int64_t>(m.r) * p.q_ss + static_cast<int64_t>(m.h * g) * p.q_sh;
    if constexpr (!MMA) {
#pragma unroll
      for (int k = 0; k < EPL / 2; ++k) o2[k] = make_float2(0.f, 0.f);
      if constexpr (EPL == 4) {   // q row -> fp32 in the warp scratch (read back as broadcasts)
        const uint2 w = noq ? make_uint2(0u, 0u) : __ldg(reinterpret_cast<const uint2 *>(qg) + lane);
        st_shared_v4f(my_scr + lane * 16, bf16lo(w.x), bf16hi(w.x), bf16lo(w.y), bf16hi(w.y));
      } else {
        const uint32_t w = noq ? 0u : __ldg(reinterpret_cast<const uint32_t *>(qg) + lane);
        st_shared_v2f(my_scr + lane * 8, bf16lo(w), bf16hi(w));
      }
      __syncwarp();
    } else {
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int n = 0; n < NT; ++n) oacc[mt][n][0] = oacc[mt][n][1] = oacc[mt][n][2] = oacc[mt][n][3] = 0.f;
      // B = Q^T (k = d, n = head): b0 = Q[head lane/4][d (lane%4)*2 ..], b1 = d + 8
#pragma unroll
      for (int n = 0; n < NT; ++n) {
        const int head = n * 8 + (lane >> 2);
        const bool ok = !noq && head < g;
        const uint32_t *qh = reinterpret_cast<const uint32_t *>(qg + static_cast<int64_t>(ok ? head : 0) * p.q_sh) + (lane & 3);
#pragma unroll
        for (int ks = 0; ks < MT; ++ks) {
          qb[ks][n][0] = ok ? __ldg(qh + ks * 8) : 0u;
          qb[ks][n][1] = ok ? __ldg(qh + ks * 8 + 4) : 0u;
        }
      }
    }
  };

  // Zero V rows outside [lo, hi) of one chunk (whole 128-byte rows, so the
  // swizzle does not matter), then make the stores visible to the warp.
  auto zero_dead_rows = [&](uint32_t sv, int lo, int hi) {
    for (int idx = lane; idx < 16 * G::HALVES * 8; idx += 32) {
      const int row = idx / (G::HALVES * 8), rest = idx - row * (G::HALVES * 8);
      if (row < lo || row >= hi)
        sts128_zero(sv + (rest >> 3) * G::HALF_BYTES + row * 128 + (rest & 7) * 16);
    }
    __syncwarp();
  };

  // One chunk: loads are placed right before their use, and the slot is handed
  // back to the issuer (`release`) as soon as both tiles sit in registers.
  // combined K|V boxes land in address order: V first when the V pool lies below K
  const uint32_t k_off = p.kv_mode == 2 ? G::KV_BYTES : 0u, v_off = G::KV_BYTES - k_off;
  auto consume = [&](uint32_t s0, int lo, int hi, auto &&release) {
    const uint32_t sk = s0 + k_off, sv = s0 + v_off;
    if (lo > 0 || hi < 16) zero_dead_rows(sv, lo, hi);   // P = 0 must never meet NaN (Q10)
    if constexpr (!MMA) {
      // ---- s_t = q.k_t : lane = (token t, half hf of d); q from the warp scratch
      const int t = lane & 15, hf = lane >> 4;
      const uint32_t krow = sk + (D == 128 ? hf * G::HALF_BYTES : 0) + t * 128;
      const int cbase = (D == 128) ? 0 : hf * 4;
      uint4 kw[NCH];
#pragma unroll
      for (int cc = 0; cc < NCH; ++cc) kw[cc] = lds128(krow + (((cbase + cc) ^ (t & 7)) << 4));
      uint32_t vcol;
      if constexpr (D == 128) vcol = sv + (lane >> 4) * G::HALF_BYTES + (lane & 1) * 8;
      else vcol = sv + (lane & 3) * 4;
      const int c = (D == 128) ? ((lane & 15) >> 1) : (lane >> 2);
      uint32_t vw[16][EPL / 2];
#pragma unroll
      for (int tt = 0; tt < 16; ++tt) {
        if constexpr (EPL == 4) {
          const uint2 w = lds64(vcol + swz(tt, c));
          vw[tt][0] = w.x;
          vw[tt][1] = w.y;
        } else {
          vw[tt][0] = lds32(vcol + swz(tt, c));
        }
      }
      release();
      float2 acc0 = make_float2(0.f, 0.f), acc1 = make_float2(0.f, 0.f);
#pragma unroll
      for (int cc = 0; cc < NCH; ++cc) {
        const uint32_t qa = my_scr + (hf * (D / 2) + cc * 8) * 4;
        const uint4 q0 = lds128(qa), q1 = lds128(qa + 16);
        const uint4 w = kw[cc];
        acc0 = __ffma2_rn(make_float2(__uint_as_float(q0.x), __uint_as_float(q0.y)),
                          make_float2(bf16lo(w.x), bf16hi(w.x)), acc0);
        acc1 = __ffma2_rn(make_float2(__uint_as_float(q0.z), __uint_as_float(q0.w)),
                          make_float2(bf16lo(w.y), bf16hi(w.y)), acc1);
        acc0 = __ffma2_rn(make_float2(__uint_as_float(q1.x), __uint_as_float(q1.y)),
                          make_float2(bf16lo(w.z), bf16hi(w.z)), acc0);
        acc1 = __ffma2_rn(make_float2(__uint_as_float(q1.z), __uint_as_float(q1.w)),
                          make_float2(bf16lo(w.w), bf16hi(w.w)), acc1);
      }
      float dot = (acc0.x + acc0.y) + (acc1.x + acc1.y);
      dot += __shfl_xor_sync(FULL, dot, 16);
      const float sc = (t >= lo && t < hi) ? dot * p.scale_log2 : -INFINITY;
      float mx = sc;
#pragma unroll
      for (int o = 8; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, o));
      const float mnew = fmaxf(mrun[0][0], mx);
      const float alpha = ex2(mrun[0][0] - mnew);
      const float pr = ex2(sc - mnew);
      lrun[0][0] = lrun[0][0] * alpha + (hf == 0 ? pr : 0.f);
      mrun[0][0] = mnew;
      // ---- o = alpha * o + sum_t p_t v_t  (p broadcast through the scratch)
      if (lane < 16) st_shared_f32(my_scr + 512 + lane * 4, pr);
      __syncwarp();
      const float2 a2 = make_float2(alpha, alpha);
#pragma unroll
      for (int k = 0; k < EPL / 2; ++k) o2[k] = __fmul2_rn(o2[k], a2);
#pragma unroll
      for (int t4 = 0; t4 < 4; ++t4) {
        const uint4 pw4 = lds128(my_scr + 512 + t4 * 16);
        const float pt[4] = {__uint_as_float(pw4.x), __uint_as_float(pw4.y), __uint_as_float(pw4.z),
                             __uint_as_float(pw4.w)};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 pp = make_float2(pt[i], pt[i]);
#pragma unroll
          for (int k = 0; k < EPL / 2; ++k)
            o2[k] = __ffma2_rn(pp, make_float2(bf16lo(vw[t4 * 4 + i][k]), bf16hi(vw[t4 * 4 + i][k])), o2[k]);
        }
      }
    } else {
      const int mi = lane >> 3;
      // ---- S^T = K . Q^T : rows = 16 tokens, cols = 8 heads per tile
      float sa[NT][4], sb[NT][4];
#pragma unroll
      for (int n = 0; n < NT; ++n)
#pragma unroll
        for (int j = 0; j < 4; ++j) sa[n][j] = sb[n][j] = 0.f;
#pragma unroll
      for (int ks = 0; ks < MT; ++ks) {
        // A = K (16 tokens x 16 d): matrices (t0-7,d0-7) (t8-15,d0-7) (t0-7,d8-15) (t8-15,d8-15)
        const int tok = (mi & 1) * 8 + (lane & 7), de = ks * 16 + (mi >> 1) * 8;
        uint32_t a0, a1, a2, a3;
        ldsm_x4(sk + (de >> 6) * G::HALF_BYTES + swz(tok, (de & 63) >> 3), a0, a1, a2, a3);
#pragma unroll
        for (int n = 0; n < NT; ++n) {
          float(&acc)[4] = (ks & 1) ? sb[n] : sa[n];   // two independent MMA chains
          mma_bf16_16816(acc, a0, a1, a2, a3, qb[ks][n][0], qb[ks][n][1]);
        }
      }
      // A = V^T (16 d x 16 tokens per d tile) via ldmatrix.trans of V rows, then free the slot
      uint32_t va[MT][4];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        const int tok = (mi >> 1) * 8 + (lane & 7), de = mt * 16 + (mi & 1) * 8;
        ldsm_x4_t(sv + (de >> 6) * G::HALF_BYTES + swz(tok, (de & 63) >> 3), va[mt][0], va[mt][1],
                  va[mt][2], va[mt][3]);
      }
      release();
      const int t0 = lane >> 2, t1 = t0 + 8;
      const bool ok0 = t0 >= lo && t0 < hi, ok1 = t1 >= lo && t1 < hi;
      // Lazy reference maximum (log2 domain), as in the planned kernel: the common chunk
      // exponentiates against the running reference (p <= 2^8); the cross-lane max, the
      // correction exponential and the O rescale run only when a live score passes the
      // reference by more than 8 (a segment's first chunk, rarely after).
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
          // P^T -> scratch as P[head][token] (row stride 48 B: conflict-free ldmatrix)
          const int head = n * 8 + (lane & 3) * 2 + j;
          st_shared_bf16(my_scr + head * 48 + t0 * 2, p0);
          st_shared_bf16(my_scr + head * 48 + t1 * 2, p1);
        }
      __syncwarp();
      // B = P^T (k = token, n = head): ldmatrix of P rows (heads) x 8 tokens
      uint32_t pb[NT][2];
      if constexpr (NT == 1) {
        const int r8 = lane & 7, hi8 = (lane >> 3) & 1;
        ldsm_x2(my_scr + r8 * 48 + hi8 * 16, pb[0][0], pb[0][1]);
      } else {
        const int r8 = lane & 7, hi8 = (lane >> 3) & 1, nn = lane >> 4;
        ldsm_x4(my_scr + (nn * 8 + r8) * 48 + hi8 * 16, pb[0][0], pb[0][1], pb[1][0], pb[1][1]);
      }
      // ---- O^T += V^T . P^T
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int n = 0; n < NT; ++n)
          mma_bf16_16816(oacc[mt][n], va[mt][0], va[mt][1], va[mt][2], va[mt][3], pb[n][0], pb[n][1]);
    }
  };

  auto end_unit = [&](const SlotMeta &m) {
    const int r = m.r, h = m.h, u = m.u;
    if constexpr (!MMA) {
      float l0 = lrun[0][0];
#pragma unroll
      for (int o = 16; o; o >>= 1) l0 += __shfl_xor_sync(FULL, l0, o);
      const int e0 = lane * EPL;
      if (m.nsplit == 1) {
        const float inv = l0 > 0.f ? 1.f / l0 : 0.f;
        uint16_t *o = p.out + static_cast<int64_t>(r) * p.o_ss + static_cast<int64_t>(h) * p.o_sh + e0;
        if constexpr (EPL == 4) {
          uint2 w;
          w.x = pack_bf16(o2[0].x * inv, o2[0].y * inv);
          w.y = pack_bf16(o2[1].x * inv, o2[1].y * inv);
          *reinterpret_cast<uint2 *>(o) = w;
        } else {
          *reinterpret_cast<uint32_t *>(o) = pack_bf16(o2[0].x * inv, o2[0].y * inv);
        }
        return;
      }
      float *po = p.part_o + static_cast<int64_t>(u) * D + e0;   // g == 1
      if constexpr (EPL == 4)
        *reinterpret_cast<float4 *>(po) = make_float4(o2[0].x, o2[0].y, o2[1].x, o2[1].y);
      else
        *reinterpret_cast<float2 *>(po) = o2[0];
      if (lane == 0)
        *reinterpret_cast<float2 *>(p.part_ml + static_cast<int64_t>(u) * 2) = make_float2(mrun[0][0], l0);
    } else {
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
      const bool direct = m.nsplit == 1;
#pragma unroll
      for (int n = 0; n < NT; ++n)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int head = n * 8 + (lane & 3) * 2 + j;
          if (head >= g) continue;
          if (direct) {
            const float inv = lsum[n][j] > 0.f ? 1.f / lsum[n][j] : 0.f;
            uint16_t *o = p.out + static_cast<int64_t>(r) * p.o_ss + static_cast<int64_t>(h * g + head) * p.o_sh;
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
              const __nv_bfloat16 b0 = __float2bfloat16_rn(oacc[mt][n][j] * inv);
              const __nv_bfloat16 b1 = __float2bfloat16_rn(oacc[mt][n][2 + j] * inv);
              o[mt * 16 + d0] = *reinterpret_cast<const uint16_t *>(&b0);
              o[mt * 16 + d0 + 8] = *reinterpret_cast<const uint16_t *>(&b1);
            }
          } else {
            float *po = p.part_o + (static_cast<int64_t>(u) * g + head) * D;
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
              po[mt * 16 + d0] = oacc[mt][n][j];
              po[mt * 16 + d0 + 8] = oacc[mt][n][2 + j];
            }
            if (d0 == 0)
              *reinterpret_cast<float2 *>(p.part_ml + (static_cast<int64_t>(u) * g + head) * 2) =
                  make_float2(mrun[n][j], lsum[n][j]);
          }
        }
      if (direct) return;
    }
    // Split partial written.  Fused merge (default): the warp that completes the
    // LAST split of (r, h) merges all of them in split order right here, while
    // other warps keep streaming -- no second kernel on the critical path.
    // Release/acquire through the per-(r, h) arrival counter (threadfence +
    // atomic, the classic last-block pattern); the counter is reset by the
    // merging warp, so the workspace stays clean for the next call.  Otherwise
    // bkv merge_kernel (next on the stream) combines the splits.
    if (p.fused_merge) {
      __syncwarp();      // every lane's partial stores precede lane 0's arrival, which
      int last = 0;      // releases them (and acquires the other splits') at gpu scope
      if (lane == 0) {
        int old;
        asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;"
                     : "=r"(old) : "l"(p.merge_cnt + r * H + h) : "memory");
        last = old == m.nsplit - 1;
      }
      last = __shfl_sync(FULL, last, 0);
      if (last) {
        const int qq = u / H;
        int k = 0;
        while (k < kBuckets - 1 && qq >= plan.base[k + 1]) ++k;
        const int u0 = (plan.base[k] + Pre[k * (p.B + 1) + r]) * H + h;
        if (g <= 8 && m.nsplit * g <= 128)
          merge_group<D>(p, u0, m.nsplit, r, h, lane, my_scr);
        else
          for (int head = 0; head < g; ++head) merge_row<D, true>(p, u0, m.nsplit, r, h, head, lane, u0, H);
        if (lane == 0) p.merge_cnt[r * H + h] = 0;
      }
    }
  };

  // ------------------------------------------------------------- main loop
  int issued = 0;
  for (; issued < S; ++issued) {
    SlotMeta m;
    int blk, cs;
    if (!next_chunk(m, blk, cs)) break;
    issue(issued, m, blk, cs);
  }
  long long prof[6] = {0, 0, 0, 0, 0, 0};   // dev (BKV_TRACE): cycles wait/begin/consume/issue/end, chunks
  const bool profiling = kDevTrace && p.trace != nullptr;
  int slot = 0;
  uint32_t phase = 0;
  for (int seq = 0; seq < issued; ++seq) {
    __syncwarp();
    const int4 mw0 = reinterpret_cast<const int4 *>(metas + slot)[0];
    const int4 mw1 = reinterpret_cast<const int4 *>(metas + slot)[1];
    const SlotMeta m{mw0.x, mw0.y, mw0.z, mw0.w, mw1.x, mw1.y, mw1.z, mw1.w};
    const long long c0 = profiling ? clock64() : 0;
    mbar_wait(my_bars + 8 * slot, phase);
    const long long c1 = profiling ? clock64() : 0;
    if (m.flags & F_FIRST) {
      trace(3, m.u);
      begin_unit(m);
    }
    if (m.flags & F_NEW) {
      // The tile was loaded before the token existed: patch its row (swizzled)
      // from the patch area, and store the row into the pool (the append).
      constexpr int TPR = D / 8;   // 16-byte pieces per row
      const int which = lane >> 4, pc = lane & 15, slot_new = (m.flags >> 8) & 0xff;
      if (pc < TPR) {
        const uint4 v = lds128(my_patch + slot * 512 + which * 2 * D + pc * 16);
        const uint32_t tile = my_slots + slot * G::SLOT_BYTES + (which ? v_off : k_off);
        st_shared_v4(tile + (pc >> 3) * G::HALF_BYTES + swz(slot_new & 15, pc & 7), v);
      }
      if (lane == 0) {   // pool rows: async bulk stores straight from the patch area
        const int64_t off = static_cast<int64_t>(m.aux) * p.pool_sb + static_cast<int64_t>(m.h) * p.pool_sh +
                            static_cast<int64_t>(slot_new) * p.pool_ss;
        bulk_store(p.k_pool + off, my_patch + slot * 512, 2 * D);
        bulk_store(p.v_pool + off, my_patch + slot * 512 + 2 * D, 2 * D);
        bulk_commit();
      }
      __syncwarp();
    }
    const long long c2 = profiling ? clock64() : 0;
    long long ci0 = 0, ci1 = 0;
    // refill this slot with the warp's next chunk (after our reads of it)
    auto release = [&]() {
      if (profiling) ci0 = clock64();
      __syncwarp();
      if (m.lo > 0 || m.hi < 16 || (m.flags & F_NEW))   // our generic smem writes precede
        fence_proxy_async_smem();                       // the next async (TMA) writes
      SlotMeta mn;
      int blk, cs;
      if (next_chunk(mn, blk, cs)) {
        issue(slot, mn, blk, cs);
        ++issued;
      }
      if (profiling) ci1 = clock64();
    };
    if (!(m.flags & F_NOKV) && !(p.debug_flags & 1)) {
      consume(my_slots + slot * G::SLOT_BYTES, m.lo, m.hi, release);
    } else {
      release();
    }
    const long long c3 = profiling ? clock64() : 0;
    if (m.flags & F_LAST) {
      end_unit(m);
      trace(4, m.u);
    }
    if (profiling) {
      const long long c4 = clock64();
      prof[0] += c1 - c0;
      prof[1] += c2 - c1;
      prof[2] += (c3 - c2) - (ci1 - ci0);
      prof[3] += ci1 - ci0;
      prof[4] += c4 - c3;
      prof[5] += 1;
    }
    if (++slot == S) {
      slot = 0;
      phase ^= 1u;
    }
  }
  if (p.k_new != nullptr && lane == 0) bulk_wait_all();   // pool rows written before exit
  if (p.fused_merge) {   // no merge kernel follows: the last CTA to exit re-arms the unit counter
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(p.sched + 1, 1) == static_cast<int>(gridDim.x) - 1) {
        p.sched[0] = 0;
        p.sched[1] = 0;
        __threadfence();
      }
    }
  }
  if (profiling)
    for (int k = 0; k < 6; ++k) trace(8 + k, static_cast<int>(min(prof[k], (long long)0x7fffffff)));

  trace(6, -1);
}

// Split merge, a second, stream-ordered kernel: one warp
// per (request, kv head, q head).  Requests with one split were written by the
// decode kernel directly; for the others the fp32 (m, l, o) partials of all
// splits are combined in split order -- M = max m_s, L = sum l_s 2^(m_s - M),
// O = sum o_s 2^(m_s - M) / L -- so the result is deterministic.  CTA 0 of the
// decode kernel publishes (first split slot, split count) per request, so a
// row's dependent chain is: that one load, all its partial loads (issued
// together for <= kFastSplits splits), the store.  Being
// stream-ordered after the decode kernel, it needs no atomics or fences; it
// also re-arms the decode kernel's unit counter for the next call.
template <int D>
__global__ void __launch_bounds__(256) merge_kernel(const DecodeParams p) {
  constexpr int EPL = D / 32;
  if (p.pdl) {
    // the next decode call's CTAs may start their seq_lens-only prologue as
    // SMs free up; they wait for this grid before touching anything else
    if (!(p.debug_flags & 32)) asm volatile("griddepcontrol.launch_dependents;");
    asm volatile("griddepcontrol.wait;" ::: "memory");   // decode results complete
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) p.sched[0] = 0;
  const int lane = threadIdx.x & 31;
  const int wid = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int H = p.H, g = p.g;
  if (wid >= p.B * H * g) return;   // one warp per (request, kv head, q head of the group)
  const int rh = wid / g, row1 = wid - rh * g;
  const int r = rh / H, h = rh - r * H;
  const int2 mp = reinterpret_cast<const int2 *>(p.plan_out + 16)[r];
  const int sk = p.plan_out[7];
  const int64_t off = static_cast<int64_t>(r) * p.o_ss + static_cast<int64_t>(h * g + row1) * p.o_sh + lane * EPL;
  int ns, u0, u_first, ustride;
  if (sk) {
    // stream-K plan: mp = (blocks of the requests before r, r's blocks); warp range w
    // covers flattened blocks [w * per, (w + 1) * per); a row cut across ranges w0..w1
    // left its pieces in slot 2 w + 0 (the range's first segment) or 2 w + 1 (its last)
    const int per = p.plan_out[0], nb = mp.y;
    if (nb == 0) {   // empty context (reading Q8): zeros; no range ever touched the row
      if constexpr (EPL == 4) {
        *reinterpret_cast<uint2 *>(p.out + off) = make_uint2(0u, 0u);
        peer_put8(p, off, make_uint2(0u, 0u));
      } else {
        *reinterpret_cast<uint32_t *>(p.out + off) = 0u;
        peer_put4(p, off, 0u);
      }
      return;
    }
    const int S = H * mp.x + h * nb;   // small problems only: fits in int
    const int w0 = S / per, w1 = (S + nb - 1) / per;
    ns = w1 - w0 + 1;
    u0 = 2 * w0;
    u_first = 2 * w0 + (S == w0 * per ? 0 : 1);
    ustride = 2;
  } else {
    // split plan: (first split slot, splits); all splits of (r, h) are consecutive
    // split slots of r's bucket: u = (slot0 + s) * H + h
    ns = mp.y;
    u0 = mp.x * H + h;
    u_first = u0;
    ustride = H;
  }
  if (ns <= 1) {
    // single split: the decode kernel wrote the local row; forward it to the
    // peers' outputs (fused reassembly) with 16-byte stores
    if (p.n_peers > 0) {
      if constexpr (EPL == 4) {
        const uint2 w = *reinterpret_cast<const uint2 *>(p.out + off);
        peer_put8(p, off, w);
      } else {
        const uint32_t w = *reinterpret_cast<const uint32_t *>(p.out + off);
        peer_put4(p, off, w);
      }
    }
    return;
  }
  merge_row<D, false>(p, u0, ns, r, h, row1, lane, u_first, ustride);
}

// ----------------------------------------------------------------- host
// g = 1 runs on the tensor-core kernel too (one useful n column of 8, but half
// the instructions per chunk of the CUDA-core kernel: no bf16 unpacking; measured
// opt13b TP1 88.8% -> 92.7% of HBM peak).  BKV_MHA_CUDA_CORES=1 (dev) keeps the
// CUDA-core kernel selectable.
static bool mha_on_mma() { return dev_switches().mha_cuda_cores == 0; }

cudaError_t decode_config(int head_dim, int group, int num_seqs, DecodeLaunch *cfg, int *slots,
                          int *q_bytes) {
  DevProps dp;
  cudaError_t e = dev_props(&dp);
  if (e != cudaSuccess) return e;
  const DevSwitches &sw = dev_switches();
  int S = sw.slots;
  const int slot_bytes = 2 * (head_dim / 64) * 2048;
  const int qb = 0;   // q is read from global (L2-prefetched), no shared-memory ring
  auto need = [&](int w, int s) {
    return 1024 + w * s * slot_bytes + w * s * (int)(sizeof(int) * 8) + w * s * 8 + w * 1024 + w * s * 512 +
           4 * (num_seqs + 1) * (int)sizeof(int) + 2 * ((num_seqs + 3) & ~3) * 4 + 256;
  };
  const bool mma = group > 1 || mha_on_mma();
  int W = sw.warps > 0 ? sw.warps : (mma ? 8 : 12);   // measured best: MMA kernels 8, CUDA-core MHA 12
  W = std::min(W, mma ? 8 : 12);                       // = the kernels' __launch_bounds__
  while (W > 4 && need(W, S) > dp.smem_optin - 1024) W -= 4;
  while (S > 1 && need(W, S) > dp.smem_optin - 1024) --S;
  cfg->grid = dp.sms * sw.ctas_per_sm;
  cfg->warps = W;
  cfg->smem_bytes = need(W, S);
  *slots = S;
  *q_bytes = qb;
  return cudaSuccess;
}

int decode_target_units(const DecodeLaunch &cfg) {
  return dev_switches().units_per_warp * cfg.grid * cfg.warps;
}

int decode_min_split(int group) {
  const int ms = dev_switches().min_split;
  return ms >= 0 ? ms : (group > 1 || mha_on_mma() ? 16 : 4);
}

template <int D, int KIND>
static cudaError_t launch_t(const CUtensorMap &tmK, const CUtensorMap &tmV, const DecodeParams &p,
                            const DecodeLaunch &cfg, cudaStream_t s) {
  {
    cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void *>(decode_kernel<D, KIND>), cfg.smem_bytes);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t lc = {};
  cudaLaunchAttribute attr[1];
  lc.gridDim = dim3(cfg.grid);
  lc.blockDim = dim3(cfg.warps * 32);
  lc.dynamicSmemBytes = cfg.smem_bytes;
  lc.stream = s;
  if (p.pdl) {   // programmatic dependent launch: the prologue overlaps the previous kernel
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
  }
  cudaError_t e = cudaLaunchKernelEx(&lc, decode_kernel<D, KIND>, tmK, tmV, p);
  if (e != cudaSuccess) return e;
  if (p.fused_merge) return cudaGetLastError();   // merged in-kernel, counter re-armed by the last CTA
  // one warp per (request, kv head, q head): measured faster than one warp per
  // (request, kv head) covering the whole group with merge_group (Llama-70B TP1
  // 114 vs 124 us, TP8 26 vs 45 us per layer)
  const int warps = p.B * p.H * p.g;
  cudaLaunchConfig_t lm = {};
  const int mw = std::max(1, std::min(8, dev_switches().merge_warps));   // warps per merge CTA
  lm.gridDim = dim3((p.debug_flags & 2) ? 1 : (warps + mw - 1) / mw);   // dev: 2 = re-arm only (times the merge)
  lm.blockDim = dim3(32 * mw);
  lm.stream = s;
  if (p.pdl) {
    lm.attrs = attr;
    lm.numAttrs = 1;
  }
  e = cudaLaunchKernelEx(&lm, merge_kernel<D>, p);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// Cross-rank completion signal for the fused reassembly.
// Thread k publishes "my slice of this step is in your output" to peer k
// (release, system scope, after the stream-ordered merge kernel completed) and
// waits for peer k's flag in its own pad (acquire).  The epoch is a device
// counter bumped once per call, so CUDA-graph replays need no host update.
// A bounded spin (timeout_ns of %globaltimer) reports through *err instead of
// hanging the GPU.
__global__ void peer_barrier_kernel(PeerBarrierParams p) {
  __shared__ uint32_t epoch_s;
  if (threadIdx.x == 0) {
    epoch_s = *p.counter + 1;
    *p.counter = epoch_s;
  }
  __syncthreads();
  const uint32_t epoch = epoch_s;
  const int k = threadIdx.x;
  if (k >= p.n) return;
  // outputs may have been stored through a multicast alias (BKV_FLAG_PEER_MULTICAST):
  // order those with the unicast accesses that follow, then publish system-wide
  asm volatile("fence.proxy.alias;" ::: "memory");
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p.pads[k] + p.rank), "r"(epoch) : "memory");
  unsigned long long t0;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  const uint32_t *mine = p.pads[p.rank] + k;
  for (;;) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
    if (static_cast<int32_t>(v - epoch) >= 0) break;
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    if (t - t0 > p.timeout_ns) {
      atomicExch(p.err, 1u);
      break;
    }
  }
}

cudaError_t launch_peer_barrier(const PeerBarrierParams &p, cudaStream_t s) {
  peer_barrier_kernel<<<1, 32, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_decode(const CUtensorMap &tmK, const CUtensorMap &tmV, const DecodeParams &p,
                          int head_dim, const DecodeLaunch &cfg, cudaStream_t s) {
  const int kind = p.g == 1 && !mha_on_mma() ? 0 : (p.g <= 8 ? 1 : 2);
  if (head_dim == 128) {
    if (kind == 0) return launch_t<128, 0>(tmK, tmV, p, cfg, s);
    if (kind == 1) return launch_t<128, 1>(tmK, tmV, p, cfg, s);
    return launch_t<128, 2>(tmK, tmV, p, cfg, s);
  }
  if (kind == 0) return launch_t<64, 0>(tmK, tmV, p, cfg, s);
  if (kind == 1) return launch_t<64, 1>(tmK, tmV, p, cfg, s);
  return launch_t<64, 2>(tmK, tmV, p, cfg, s);
}

}  // namespace bkv
