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
// Design (B200):
//  * Persistent grid, one CTA per SM, W independent warps per CTA.  Each warp
//    is its own producer: lane 0 streams 16-slot "chunks" (K and V tile of one
//    (block, kv head), 2*d*32 bytes) through a private S-deep ring of
//    128B-swizzled shared-memory slots with 4-D TMA tensor loads and mbarrier
//    completion, so S*8 KiB per warp are in flight while it computes.
//  * Work units = (request, kv head, split of <= P blocks), pulled from a
//    global atomic counter; full-size splits are enumerated before the
//    remainders (largest first).  P is chosen in-kernel from sum(ceil(L/bs))
//    so the whole grid gets work (split-K only as needed).
//  * MHA (g = 1): CUDA-core fp32 dot products, lanes = (token, half of d).
//  * GQA (g >= 2): the g query heads of a kv head form the M rows of a bf16
//    mma.sync m16n8k16 tile: S = Q.K^T (K via ldmatrix), online softmax on the
//    accumulator fragments, O += P.V with P re-used from registers as the A
//    operand and V via ldmatrix.trans.
//  * A unit's output is written directly when the request has one split;
//    otherwise fp32 (m, l, o) partials go to the workspace and the last split
//    to arrive merges all of them in split order (deterministic).
//  * NaN hygiene (reading Q10): dead slots are never combined arithmetically:
//    their scores are selected to -inf and (MMA path) their V rows are zeroed
//    in shared memory before P.V.
#include <math.h>

#include "bkv_internal.h"
#include "bkv_ptx.cuh"

namespace bkv {

enum : int { F_FIRST = 1, F_LAST = 2, F_NOKV = 4, F_NOQ = 8 };

struct SlotMeta {
  int u, r, h, nsplit;
  int lo, hi, flags, qidx;
};

struct Plan {
  int P;   // blocks per full split
  int FB;  // full splits over all requests
  int RB;  // remainder splits over all requests
  int U;   // units = (FB + RB) * H
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

// Split plan, computed identically by every CTA from seq_lens.
__device__ void compute_plan(const DecodeParams &p, int *F, int *R, Plan *plan) {
  __shared__ long long red_ll[32];
  __shared__ int2 red2[32];
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5,
            nw = nt >> 5;
  long long local = 0;
  for (int r = tid; r < p.B; r += nt) local += nblocks_of(__ldg(p.seq_lens + r), p.bs);
#pragma unroll
  for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if (lane == 0) red_ll[warp] = local;
  __syncthreads();
  long long T = 0;
  for (int w = 0; w < nw; ++w) T += red_ll[w];
  const long long work = T * p.H;
  long long Pll = (work + p.target_units - 1) / p.target_units;
  if (Pll < p.min_split) Pll = p.min_split;
  const int P = static_cast<int>(Pll);
  // exclusive scans of full_r = nb/P and rem_r = (nb % P != 0 || nb == 0)
  const int per = (p.B + nt - 1) / nt;
  const int r0 = min(p.B, tid * per), r1 = min(p.B, r0 + per);
  int fs = 0, rs = 0;
  for (int r = r0; r < r1; ++r) {
    const int nb = nblocks_of(__ldg(p.seq_lens + r), p.bs);
    fs += nb / P;
    rs += (nb % P != 0 || nb == 0) ? 1 : 0;
  }
  int fi = fs, ri = rs;  // inclusive warp scan
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int fu = __shfl_up_sync(0xffffffffu, fi, o), ru = __shfl_up_sync(0xffffffffu, ri, o);
    if (lane >= o) {
      fi += fu;
      ri += ru;
    }
  }
  if (lane == 31) red2[warp] = make_int2(fi, ri);
  __syncthreads();
  int fo = fi - fs, ro = ri - rs;
  for (int w = 0; w < warp; ++w) {
    fo += red2[w].x;
    ro += red2[w].y;
  }
  for (int r = r0; r < r1; ++r) {
    F[r] = fo;
    R[r] = ro;
    const int nb = nblocks_of(__ldg(p.seq_lens + r), p.bs);
    fo += nb / P;
    ro += (nb % P != 0 || nb == 0) ? 1 : 0;
  }
  if (tid == nt - 1) {
    int ft = 0, rt = 0;
    for (int w = 0; w < nw; ++w) {
      ft += red2[w].x;
      rt += red2[w].y;
    }
    F[p.B] = ft;
    R[p.B] = rt;
    plan->P = P;
    plan->FB = ft;
    plan->RB = rt;
    plan->U = (ft + rt) * p.H;
  }
  __syncthreads();
}

// KIND 0: MHA on CUDA cores; 1: MMA with g <= 8; 2: MMA with 8 < g <= 16.
template <int D, int KIND>
__global__ void __launch_bounds__(256, 1)
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
  const uint32_t q_base = slots_base + W * S * G::SLOT_BYTES;
  uint8_t *meta_g = gbase + (q_base - base) + W * (S + 1) * p.q_bytes;
  SlotMeta *metas = reinterpret_cast<SlotMeta *>(meta_g) + warp * S;
  uint64_t *bars_g = reinterpret_cast<uint64_t *>(meta_g + W * S * sizeof(SlotMeta));
  uint8_t *scratch_g = reinterpret_cast<uint8_t *>(bars_g + W * S);   // W x 64 B
  const uint32_t my_p = smem_u32(scratch_g + warp * 64);
  int *F = reinterpret_cast<int *>(scratch_g + W * 64);
  int *R = F + (p.B + 1);

  if (threadIdx.x == 0) {
    prefetch_tmap(&tmK);
    prefetch_tmap(&tmV);
  }
  compute_plan(p, F, R, &plan);
  const int P = plan.P, FB = plan.FB, U = plan.U;

  const uint32_t my_slots = slots_base + warp * S * G::SLOT_BYTES;
  const uint32_t my_q = q_base + warp * (S + 1) * p.q_bytes;
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
  int u_next = 0;
  if (lane == 0) u_next = atomicAdd(p.sched, 1);
  bool is_active = false, is_done = false, is_first = false;
  int is_u = 0, is_r = 0, is_h = 0, is_ns = 0, is_L = 0, is_e = 0, is_e1 = 0, is_c = 0;
  int is_wb = 0, bt_w = 0, dir_w = 0, is_qidx = S;  // first unit -> q-ring entry 0

  // Produce the next chunk of this warp's work stream (warp-collective).
  auto next_chunk = [&](SlotMeta &m, int &blk, int &csub) -> bool {
    if (!is_active) {
      if (is_done) return false;
      const int u = __shfl_sync(FULL, u_next, 0);
      if (u >= U) {
        is_done = true;
        return false;
      }
      if (lane == 0) u_next = atomicAdd(p.sched, 1);  // prefetch the next grab
      const int h = u % H, qq = u / H;
      int r, e0, e1;
      if (qq < FB) {
        r = search_le(F, p.B, qq);
        e0 = (qq - F[r]) * P;
        e1 = e0 + P;
      } else {
        r = search_le(R, p.B, qq - FB);
        e0 = (F[r + 1] - F[r]) * P;
        e1 = nblocks_of(__ldg(p.seq_lens + r), bs);
      }
      is_u = u;
      is_r = r;
      is_h = h;
      is_L = __ldg(p.seq_lens + r);
      is_ns = (F[r + 1] - F[r]) + (R[r + 1] - R[r]);
      is_qidx = (is_qidx == S) ? 0 : is_qidx + 1;
      is_e = e0;
      is_e1 = e1;
      is_c = 0;
      is_wb = -(1 << 30);
      is_first = true;
      if (e0 >= e1) {  // empty context (L = 0, reading Q8): one flag-only chunk
        m = SlotMeta{u, r, h, is_ns, 0, 0, F_FIRST | F_LAST | F_NOKV | F_NOQ, is_qidx};
        blk = 0;
        csub = 0;
        return true;
      }
      is_active = true;
    }
    if (is_e - is_wb >= 32) {  // refill the block-table window (32 entries, one per lane)
      is_wb = is_e;
      const int e = is_wb + lane;
      if (e < is_e1) {
        bt_w = __ldg(p.bt + static_cast<int64_t>(is_r) * p.bt_stride + e);
        dir_w = __ldg(p.dirs + static_cast<int64_t>(is_r) * p.dir_rs +
                      static_cast<int64_t>(e) * p.dir_cs);
      }
    }
    const int idx = is_e - is_wb;
    const int b = __shfl_sync(FULL, bt_w, idx);
    const int dr = __shfl_sync(FULL, dir_w, idx);
    const int ne = min(bs, is_L - is_e * bs);       // live tokens in this block
    const int lo_s = dr ? bs - ne : 0;               // RT from the left,
    const int hi_s = dr ? bs : ne;                   //        BE from the right
    const int lo = max(lo_s - is_c * 16, 0), hi = min(hi_s - is_c * 16, 16);
    int flags = (is_first ? F_FIRST : 0) | (lo >= hi ? F_NOKV : 0);
    is_first = false;
    csub = is_c;
    blk = b;
    if (++is_c == chunks_per_block) {
      is_c = 0;
      ++is_e;
    }
    if (is_e == is_e1) {
      flags |= F_LAST;
      is_active = false;
    }
    m = SlotMeta{is_u, is_r, is_h, is_ns, lo, hi, flags, is_qidx};
    return true;
  };

  auto issue = [&](int i, const SlotMeta &m, int blk, int csub) {
    if (lane == 0) {
      metas[i] = m;
      const uint32_t bar = my_bars + 8 * i;
      const bool kv = !(m.flags & F_NOKV);
      const bool qq = (m.flags & F_FIRST) && !(m.flags & F_NOQ);
      const uint32_t bytes = (kv ? G::SLOT_BYTES : 0) + (qq ? g * D * 2 : 0);
      mbar_arrive_expect_tx(bar, bytes);
      if (kv) {
        const uint32_t dk = my_slots + i * G::SLOT_BYTES, dv = dk + G::KV_BYTES;
#pragma unroll
        for (int hr = 0; hr < G::HALVES; ++hr) {
          tma_load_4d(dk + hr * G::HALF_BYTES, &tmK, hr * 64, csub * 16, m.h, blk, bar, pol);
          tma_load_4d(dv + hr * G::HALF_BYTES, &tmV, hr * 64, csub * 16, m.h, blk, bar, pol);
        }
      }
      if (qq) {
        const uint32_t dq = my_q + m.qidx * p.q_bytes;
        for (int j = 0; j < g; ++j)
          bulk_load(dq + j * D * 2,
                    p.q + static_cast<int64_t>(m.r) * p.q_ss +
                        static_cast<int64_t>(m.h * g + j) * p.q_sh,
                    D * 2, bar);
      }
    }
  };

  // --------------------------------------------------------- consumer state
  constexpr int NCH = D / 16;  // MHA: 16-byte pieces of K per lane
  constexpr int EPL = D / 32;  // MHA: output elements per lane
  float qf[MMA ? 1 : D / 2];
  float o_mha[EPL];
  uint32_t qa[MMA ? D / 16 : 1][G16 ? 4 : 2];
  float o_mma[MMA ? D / 8 : 1][4];
  float m0 = -INFINITY, l0 = 0.f, m1 = -INFINITY, l1 = 0.f;

  auto begin_unit = [&](const SlotMeta &m) {
    m0 = m1 = -INFINITY;
    l0 = l1 = 0.f;
    const uint32_t qs = my_q + m.qidx * p.q_bytes;
    if constexpr (!MMA) {
#pragma unroll
      for (int k = 0; k < EPL; ++k) o_mha[k] = 0.f;
      if (!(m.flags & F_NOQ)) {
        const int hf = lane >> 4;
#pragma unroll
        for (int cc = 0; cc < NCH; ++cc) {
          const uint4 w = lds128(qs + (hf * (D / 2) + cc * 8) * 2);
          qf[cc * 8 + 0] = bf16lo(w.x);
          qf[cc * 8 + 1] = bf16hi(w.x);
          qf[cc * 8 + 2] = bf16lo(w.y);
          qf[cc * 8 + 3] = bf16hi(w.y);
          qf[cc * 8 + 4] = bf16lo(w.z);
          qf[cc * 8 + 5] = bf16hi(w.z);
          qf[cc * 8 + 6] = bf16lo(w.w);
          qf[cc * 8 + 7] = bf16hi(w.w);
        }
      }
    } else {
#pragma unroll
      for (int n = 0; n < D / 8; ++n) o_mma[n][0] = o_mma[n][1] = o_mma[n][2] = o_mma[n][3] = 0.f;
      const int row0 = lane >> 2, cq = (lane & 3) * 2;
      const bool noq = m.flags & F_NOQ;
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks) {
        const uint32_t a = qs + (row0 * D + ks * 16 + cq) * 2;
        const bool ok0 = !noq && row0 < g;
        qa[ks][0] = ok0 ? lds32(a) : 0u;
        qa[ks][1] = ok0 ? lds32(a + 16) : 0u;
        if constexpr (G16) {
          const bool ok1 = !noq && row0 + 8 < g;
          qa[ks][2] = ok1 ? lds32(a + 8 * D * 2) : 0u;
          qa[ks][3] = ok1 ? lds32(a + 8 * D * 2 + 16) : 0u;
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

  auto consume = [&](uint32_t sk, int lo, int hi) {
    const uint32_t sv = sk + G::KV_BYTES;
    if constexpr (!MMA) {
      // ---- S = scale * q.k for 16 tokens; lane = (token t, half hf of d)
      const int t = lane & 15, hf = lane >> 4;
      const uint32_t krow = sk + (D == 128 ? hf * G::HALF_BYTES : 0) + t * 128;
      const int cbase = (D == 128) ? 0 : hf * 4;
      float d0 = 0.f, d1 = 0.f, d2 = 0.f, d3 = 0.f;
#pragma unroll
      for (int cc = 0; cc < NCH; ++cc) {
        const uint4 w = lds128(krow + (((cbase + cc) ^ (t & 7)) << 4));
        d0 = fmaf(qf[cc * 8 + 0], bf16lo(w.x), d0);
        d1 = fmaf(qf[cc * 8 + 1], bf16hi(w.x), d1);
        d2 = fmaf(qf[cc * 8 + 2], bf16lo(w.y), d2);
        d3 = fmaf(qf[cc * 8 + 3], bf16hi(w.y), d3);
        d0 = fmaf(qf[cc * 8 + 4], bf16lo(w.z), d0);
        d1 = fmaf(qf[cc * 8 + 5], bf16hi(w.z), d1);
        d2 = fmaf(qf[cc * 8 + 6], bf16lo(w.w), d2);
        d3 = fmaf(qf[cc * 8 + 7], bf16hi(w.w), d3);
      }
      float dot = (d0 + d1) + (d2 + d3);
      dot += __shfl_xor_sync(FULL, dot, 16);
      const float s = (t >= lo && t < hi) ? dot * p.scale_log2 : -INFINITY;
      float mx = s;
#pragma unroll
      for (int o = 8; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, o));
      const float mnew = fmaxf(m0, mx);
      const float alpha = ex2(m0 - mnew);
      const float pr = ex2(s - mnew);
      l0 = l0 * alpha + (hf == 0 ? pr : 0.f);
      m0 = mnew;
#pragma unroll
      for (int k = 0; k < EPL; ++k) o_mha[k] *= alpha;
      // ---- o += p_t * v_t.  Dead rows of a partly live chunk are zeroed first
      // (p_t = 0 there, and 0 * NaN must never happen -- reading Q10); then all
      // 16 tokens are unrolled with p broadcast from shared memory.
      if (lo > 0 || hi < 16) zero_dead_rows(sv, lo, hi);
      if (lane < 16) st_shared_f32(my_p + lane * 4, pr);
      __syncwarp();
      float pt[16];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint4 w = lds128(my_p + k * 16);
        pt[4 * k + 0] = __uint_as_float(w.x);
        pt[4 * k + 1] = __uint_as_float(w.y);
        pt[4 * k + 2] = __uint_as_float(w.z);
        pt[4 * k + 3] = __uint_as_float(w.w);
      }
      uint32_t vcol;
      if constexpr (D == 128) {
        vcol = sv + (lane >> 4) * G::HALF_BYTES + (lane & 1) * 8;
      } else {
        vcol = sv + (lane & 3) * 4;
      }
      const int c = (D == 128) ? ((lane & 15) >> 1) : (lane >> 2);
#pragma unroll
      for (int tt = 0; tt < 16; ++tt) {
        const uint32_t a = vcol + swz(tt, c);
        if constexpr (D == 128) {
          const uint2 w = lds64(a);
          o_mha[0] = fmaf(pt[tt], bf16lo(w.x), o_mha[0]);
          o_mha[1] = fmaf(pt[tt], bf16hi(w.x), o_mha[1]);
          o_mha[2] = fmaf(pt[tt], bf16lo(w.y), o_mha[2]);
          o_mha[3] = fmaf(pt[tt], bf16hi(w.y), o_mha[3]);
        } else {
          const uint32_t w = lds32(a);
          o_mha[0] = fmaf(pt[tt], bf16lo(w), o_mha[0]);
          o_mha[1] = fmaf(pt[tt], bf16hi(w), o_mha[1]);
        }
      }
    } else {
      // ---- S^T tile: rows = query heads of the group, cols = 16 tokens
      float sacc[2][4];
#pragma unroll
      for (int n = 0; n < 2; ++n) sacc[n][0] = sacc[n][1] = sacc[n][2] = sacc[n][3] = 0.f;
      const int mi = lane >> 3;
      // all K fragments first (the asm loads/MMAs keep program order), then the MMAs
      uint32_t kb[D / 16][4];
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks) {
        const int tok = (mi >> 1) * 8 + (lane & 7), ke = ks * 16 + (mi & 1) * 8;
        ldsm_x4(sk + (ke >> 6) * G::HALF_BYTES + swz(tok, (ke & 63) >> 3), kb[ks][0], kb[ks][1],
                kb[ks][2], kb[ks][3]);
      }
      float sacc2[2][4];
#pragma unroll
      for (int n = 0; n < 2; ++n) sacc2[n][0] = sacc2[n][1] = sacc2[n][2] = sacc2[n][3] = 0.f;
#pragma unroll
      for (int ks = 0; ks < D / 16; ++ks) {
        const uint32_t a1 = G16 ? qa[ks][2] : 0u, a3 = G16 ? qa[ks][3] : 0u;
        float(&acc0)[4] = (ks & 1) ? sacc2[0] : sacc[0];   // two independent chains
        float(&acc1)[4] = (ks & 1) ? sacc2[1] : sacc[1];
        mma_bf16_16816(acc0, qa[ks][0], a1, qa[ks][1], a3, kb[ks][0], kb[ks][1]);
        mma_bf16_16816(acc1, qa[ks][0], a1, qa[ks][1], a3, kb[ks][2], kb[ks][3]);
      }
#pragma unroll
      for (int n = 0; n < 2; ++n)
#pragma unroll
        for (int j = 0; j < 4; ++j) sacc[n][j] += sacc2[n][j];
      const int cq = (lane & 3) * 2;
      float s0[4], s1[4];
#pragma unroll
      for (int n = 0; n < 2; ++n)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int tok = n * 8 + cq + j;
          const bool ok = tok >= lo && tok < hi;
          s0[n * 2 + j] = ok ? sacc[n][j] * p.scale_log2 : -INFINITY;
          s1[n * 2 + j] = ok ? sacc[n][2 + j] * p.scale_log2 : -INFINITY;
        }
      float mx = fmaxf(fmaxf(s0[0], s0[1]), fmaxf(s0[2], s0[3]));
      mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(FULL, mx, 2));
      const float mn0 = fmaxf(m0, mx), al0 = ex2(m0 - mn0);
      float pr0[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) pr0[k] = ex2(s0[k] - mn0);
      l0 = l0 * al0 + ((pr0[0] + pr0[1]) + (pr0[2] + pr0[3]));
      m0 = mn0;
      float pr1[4] = {0.f, 0.f, 0.f, 0.f}, al1 = 1.f;
      if constexpr (G16) {
        float mx1 = fmaxf(fmaxf(s1[0], s1[1]), fmaxf(s1[2], s1[3]));
        mx1 = fmaxf(mx1, __shfl_xor_sync(FULL, mx1, 1));
        mx1 = fmaxf(mx1, __shfl_xor_sync(FULL, mx1, 2));
        const float mn1 = fmaxf(m1, mx1);
        al1 = ex2(m1 - mn1);
#pragma unroll
        for (int k = 0; k < 4; ++k) pr1[k] = ex2(s1[k] - mn1);
        l1 = l1 * al1 + ((pr1[0] + pr1[1]) + (pr1[2] + pr1[3]));
        m1 = mn1;
      }
      (void)s1;
#pragma unroll
      for (int n = 0; n < D / 8; ++n) {
        o_mma[n][0] *= al0;
        o_mma[n][1] *= al0;
        if constexpr (G16) {
          o_mma[n][2] *= al1;
          o_mma[n][3] *= al1;
        }
      }
      const uint32_t pa0 = pack_bf16(pr0[0], pr0[1]), pa2 = pack_bf16(pr0[2], pr0[3]);
      const uint32_t pa1 = G16 ? pack_bf16(pr1[0], pr1[1]) : 0u;
      const uint32_t pa3 = G16 ? pack_bf16(pr1[2], pr1[3]) : 0u;
      // ---- zero dead V rows of a partly live chunk (P = 0 must not meet NaN)
      if (lo > 0 || hi < 16) zero_dead_rows(sv, lo, hi);
      // ---- O += P . V  (V fragments first, then the MMAs)
      uint32_t vb[D / 16][4];
#pragma unroll
      for (int nb = 0; nb < D / 16; ++nb) {
        const int tok = (mi & 1) * 8 + (lane & 7), de = nb * 16 + (mi >> 1) * 8;
        ldsm_x4_t(sv + (de >> 6) * G::HALF_BYTES + swz(tok, (de & 63) >> 3), vb[nb][0], vb[nb][1],
                  vb[nb][2], vb[nb][3]);
      }
#pragma unroll
      for (int nb = 0; nb < D / 16; ++nb) {
        mma_bf16_16816(o_mma[2 * nb], pa0, pa1, pa2, pa3, vb[nb][0], vb[nb][1]);
        mma_bf16_16816(o_mma[2 * nb + 1], pa0, pa1, pa2, pa3, vb[nb][2], vb[nb][3]);
      }
    }
  };

  // Merge all split partials of (r, h) in split order and write bf16 out rows.
  auto merge_splits = [&](const SlotMeta &m) {
    const int r = m.r, h = m.h;
    const int nfull = F[r + 1] - F[r];
    for (int row = 0; row < g; ++row) {
      float M = -INFINITY;
      for (int s = 0; s < m.nsplit; ++s) {
        const int us = s < nfull ? (F[r] + s) * H + h : (FB + R[r]) * H + h;
        M = fmaxf(M, __ldcg(p.part_ml + (static_cast<int64_t>(us) * g + row) * 2));
      }
      float Ls = 0.f, acc[EPL];
#pragma unroll
      for (int k = 0; k < EPL; ++k) acc[k] = 0.f;
      for (int s = 0; s < m.nsplit; ++s) {
        const int us = s < nfull ? (F[r] + s) * H + h : (FB + R[r]) * H + h;
        const int64_t pr = static_cast<int64_t>(us) * g + row;
        const float ms = __ldcg(p.part_ml + pr * 2), ls = __ldcg(p.part_ml + pr * 2 + 1);
        const float w = ex2(ms - M);
        Ls = fmaf(ls, w, Ls);
#pragma unroll
        for (int k = 0; k < EPL; ++k) acc[k] = fmaf(w, __ldcg(p.part_o + pr * D + lane + 32 * k), acc[k]);
      }
      const float inv = Ls > 0.f ? 1.f / Ls : 0.f;
      uint16_t *o = p.out + static_cast<int64_t>(r) * p.o_ss + static_cast<int64_t>(h * g + row) * p.o_sh;
#pragma unroll
      for (int k = 0; k < EPL; ++k) {
        const __nv_bfloat16 b = __float2bfloat16_rn(acc[k] * inv);
        o[lane + 32 * k] = *reinterpret_cast<const uint16_t *>(&b);
      }
    }
    if (lane == 0) p.counters[r * H + h] = 0;  // self-reset for the next call
  };

  auto end_unit = [&](const SlotMeta &m) {
    const int r = m.r, h = m.h, u = m.u;
    if constexpr (!MMA) {
#pragma unroll
      for (int o = 16; o; o >>= 1) l0 += __shfl_xor_sync(FULL, l0, o);
      const int e0 = lane * EPL;
      if (m.nsplit == 1) {
        const float inv = l0 > 0.f ? 1.f / l0 : 0.f;
        uint16_t *o = p.out + static_cast<int64_t>(r) * p.o_ss + static_cast<int64_t>(h) * p.o_sh + e0;
        if constexpr (EPL == 4) {
          uint2 w;
          w.x = pack_bf16(o_mha[0] * inv, o_mha[1] * inv);
          w.y = pack_bf16(o_mha[2] * inv, o_mha[3] * inv);
          *reinterpret_cast<uint2 *>(o) = w;
        } else {
          *reinterpret_cast<uint32_t *>(o) = pack_bf16(o_mha[0] * inv, o_mha[1] * inv);
        }
        return;
      }
      float *po = p.part_o + static_cast<int64_t>(u) * D + e0;   // g == 1
      if constexpr (EPL == 4)
        *reinterpret_cast<float4 *>(po) = make_float4(o_mha[0], o_mha[1], o_mha[2], o_mha[3]);
      else
        *reinterpret_cast<float2 *>(po) = make_float2(o_mha[0], o_mha[1]);
      if (lane == 0) *reinterpret_cast<float2 *>(p.part_ml + static_cast<int64_t>(u) * 2) = make_float2(m0, l0);
    } else {
      l0 += __shfl_xor_sync(FULL, l0, 1);
      l0 += __shfl_xor_sync(FULL, l0, 2);
      if constexpr (G16) {
        l1 += __shfl_xor_sync(FULL, l1, 1);
        l1 += __shfl_xor_sync(FULL, l1, 2);
      }
      const int row0 = lane >> 2, cq = (lane & 3) * 2;
      if (m.nsplit == 1) {
        const float inv0 = l0 > 0.f ? 1.f / l0 : 0.f;
        if (row0 < g) {
          uint16_t *o = p.out + static_cast<int64_t>(r) * p.o_ss + static_cast<int64_t>(h * g + row0) * p.o_sh + cq;
#pragma unroll
          for (int n = 0; n < D / 8; ++n)
            *reinterpret_cast<uint32_t *>(o + n * 8) = pack_bf16(o_mma[n][0] * inv0, o_mma[n][1] * inv0);
        }
        if constexpr (G16) {
          const float inv1 = l1 > 0.f ? 1.f / l1 : 0.f;
          if (row0 + 8 < g) {
            uint16_t *o = p.out + static_cast<int64_t>(r) * p.o_ss + static_cast<int64_t>(h * g + row0 + 8) * p.o_sh + cq;
#pragma unroll
            for (int n = 0; n < D / 8; ++n)
              *reinterpret_cast<uint32_t *>(o + n * 8) = pack_bf16(o_mma[n][2] * inv1, o_mma[n][3] * inv1);
          }
        }
        return;
      }
      if (row0 < g) {
        float *po = p.part_o + (static_cast<int64_t>(u) * g + row0) * D + cq;
#pragma unroll
        for (int n = 0; n < D / 8; ++n) *reinterpret_cast<float2 *>(po + n * 8) = make_float2(o_mma[n][0], o_mma[n][1]);
        if ((lane & 3) == 0)
          *reinterpret_cast<float2 *>(p.part_ml + (static_cast<int64_t>(u) * g + row0) * 2) = make_float2(m0, l0);
      }
      if constexpr (G16) {
        if (row0 + 8 < g) {
          float *po = p.part_o + (static_cast<int64_t>(u) * g + row0 + 8) * D + cq;
#pragma unroll
          for (int n = 0; n < D / 8; ++n) *reinterpret_cast<float2 *>(po + n * 8) = make_float2(o_mma[n][2], o_mma[n][3]);
          if ((lane & 3) == 0)
            *reinterpret_cast<float2 *>(p.part_ml + (static_cast<int64_t>(u) * g + row0 + 8) * 2) = make_float2(m1, l1);
        }
      }
    }
    // split partial written: count arrivals; the last split merges (deterministic order)
    __threadfence();
    __syncwarp();
    int prev = 0;
    if (lane == 0) prev = atomicAdd(p.counters + r * H + h, 1);
    prev = __shfl_sync(FULL, prev, 0);
    if (prev == m.nsplit - 1) {
      __threadfence();
      merge_splits(m);
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
  int slot = 0;
  uint32_t phase = 0;
  for (int seq = 0; seq < issued; ++seq) {
    __syncwarp();
    const SlotMeta m = metas[slot];
    mbar_wait(my_bars + 8 * slot, phase);
    if (m.flags & F_FIRST) begin_unit(m);
    if (!(m.flags & F_NOKV)) consume(my_slots + slot * G::SLOT_BYTES, m.lo, m.hi);
    __syncwarp();
    fence_proxy_async_smem();  // our smem reads/writes of this slot precede the TMA refill
    {
      SlotMeta mn;
      int blk, cs;
      if (next_chunk(mn, blk, cs)) {
        issue(slot, mn, blk, cs);
        ++issued;
      }
    }
    if (m.flags & F_LAST) end_unit(m);
    if (++slot == S) {
      slot = 0;
      phase ^= 1u;
    }
  }

  // ------------------------------------------------- scheduler self-reset
  __syncwarp();
  if (lane == 0) {
    __threadfence();
    const int d = atomicAdd(p.sched + 1, 1);
    if (d == p.total_warps - 1) {
      p.sched[0] = 0;
      p.sched[1] = 0;
      __threadfence();
    }
  }
}

// ----------------------------------------------------------------- host
static int env_int(const char *name, int dflt) {
  const char *s = getenv(name);
  return (s && *s) ? atoi(s) : dflt;
}

cudaError_t decode_config(int head_dim, int group, int num_seqs, DecodeLaunch *cfg, int *slots,
                          int *q_bytes) {
  int dev = 0, sms = 0, smem_optin = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) return e;
  e = cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) return e;
  const int W = env_int("BKV_WARPS", 4);
  int S = env_int("BKV_SLOTS", 4);
  const int slot_bytes = 2 * (head_dim / 64) * 2048;
  const int qb = ((group * head_dim * 2) + 127) / 128 * 128;
  auto need = [&](int s) {
    return 1024 + W * s * slot_bytes + W * (s + 1) * qb + W * s * (int)(sizeof(int) * 8) +
           W * s * 8 + W * 64 + 2 * (num_seqs + 1) * (int)sizeof(int) + 256;
  };
  while (S > 1 && need(S) > smem_optin - 1024) --S;
  cfg->grid = sms * env_int("BKV_CTAS_PER_SM", 1);
  cfg->warps = W;
  cfg->smem_bytes = need(S);
  *slots = S;
  *q_bytes = qb;
  return cudaSuccess;
}

int decode_target_units(const DecodeLaunch &cfg) {
  return env_int("BKV_UNITS_PER_WARP", 4) * cfg.grid * cfg.warps;
}

int decode_min_split(int group) { return env_int("BKV_MIN_SPLIT", group > 1 ? 16 : 4); }

template <int D, int KIND>
static cudaError_t launch_t(const CUtensorMap &tmK, const CUtensorMap &tmV, const DecodeParams &p,
                            const DecodeLaunch &cfg, cudaStream_t s) {
  static int configured = 0;  // max dynamic smem already granted to this instantiation
  if (cfg.smem_bytes > configured) {
    cudaError_t e = cudaFuncSetAttribute(decode_kernel<D, KIND>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, cfg.smem_bytes);
    if (e != cudaSuccess) return e;
    configured = cfg.smem_bytes;
  }
  decode_kernel<D, KIND><<<cfg.grid, cfg.warps * 32, cfg.smem_bytes, s>>>(tmK, tmV, p);
  return cudaGetLastError();
}

cudaError_t launch_decode(const CUtensorMap &tmK, const CUtensorMap &tmV, const DecodeParams &p,
                          int head_dim, const DecodeLaunch &cfg, cudaStream_t s) {
  const int kind = p.g == 1 ? 0 : (p.g <= 8 ? 1 : 2);
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
