// prefill_tc.cu -- mixed prefill + decode attention on the 5th-generation
// tensor cores (tcgen05.mma, TMEM accumulators) for head_dim 128
// (PAPER.md P:762-765).  Same contract as
// prefill_attention.cu: rows = (token, q head of the group) pairs, causal over
// the request's paged tokens, dense or general block maps.  The default for
// head_dim 128 (see prefill_uses_tc() in prefill_attention.cu).
//
// Persistent CTAs (one per SM) walk work items = QT consecutive 128-row query
// tiles of one (request, kv head), latest rows first (tiles aligned to the end
// of the request's rows); QT = 2 by default ("ping-pong": both tiles share every
// streamed K/V tile).  Roles, for QT = 2 (352 threads):
//   warps 0-3, 4-7  one softmax warpgroup per query tile: thread t owns row t
//              of its tile and TMEM lane t (tcgen05.ld 32x32b gives a whole
//              row to one thread: no shuffles); masks (direction + causal by
//              token index; a mask-free path for whole tiles), online
//              softmax in the log2 domain -- a speculative pass against the
//              running reference, the exact pass (row max, lazy O rescale: the
//              reference moves only when a score passes it by > 8) only when
//              needed -- writes P (bf16 pairs) back into the TMEM columns of the
//              S buffer it just read, zeroes dead V rows (group 0), runs the
//              epilogue (shared-memory staging + TMA store);
//   warp 8     K producer: walks the request's entries lane-parallel, TMA-loads
//              the item's Q, publishes each 64-key tile's chunk metadata
//              (5-slot ring, named barriers) and TMA-streams the K tile (four
//              16-slot chunks as rows of one 128B-swizzled operand) into a
//              3-stage K ring freed by the S MMAs;
//   warp 9     MMA warp + TMEM owner (one elected lane issues): per key tile,
//              for each query tile S = Q.K^T (M 128, N <= 64, K 128) into one
//              of two TMEM S buffers, then O += P.V (M 128, N 128, K 16 per
//              chunk, A = P straight from TMEM: the "TS" form) into that tile's
//              TMEM O accumulator; tcgen05.commit releases buffers and stages;
//   warp 10    V producer (same walk, V tiles, a 3-stage V ring freed by P.V).
// Operands: Q and K are K-major 128B-swizzled, V is MN-major 128B-swizzled
// -- exactly the layout the TMA boxes land in; P never leaves TMEM.
#include <math.h>

#include "bkv_internal.h"
#include "bkv_ptx.cuh"

namespace bkv {

namespace {

constexpr int kTcStages = 4;       // key-tile ring (K | V of up to 64 keys per stage)
constexpr int kTcChunks = 4;       // chunks (16 keys each) per key tile
constexpr int kTcKeys = 16 * kTcChunks;
constexpr int kTcLastFlag = 1 << 8;   // tile metadata: the item's last key tile
constexpr int kTcPatchFlag = 1 << 9;
constexpr int kLiveCap = 512;         // batches up to this many requests enumerate only the requests with rows  // tile metadata: some chunk is partly live (dead V rows to zero)
constexpr int kTcRows = 128;       // query rows per CTA = TMEM lanes

__device__ __forceinline__ uint32_t tswz(int row, int c) {
  return static_cast<uint32_t>(row * 128 + ((c ^ (row & 7)) << 4));
}

// SM100 shared-memory matrix descriptor, 128B swizzle (start, leading and
// stride byte offsets in 16-byte units; version 1).
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// instruction descriptor: bf16 x bf16 -> fp32, shape M x N, A/B major (0 K, 1 MN)
__host__ __device__ constexpr uint32_t idesc(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// Warp-collective forms: the whole (converged) warp executes them and one
// elected lane issues -- the descriptors stay warp-uniform (uniform registers),
// with no per-instruction single-lane divergence loop around the issue.
__device__ __forceinline__ void umma_commit_w(uint32_t bar) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(bar)
      : "memory");
}
// S = Q.K^T of one 64-key tile: eight K=16 steps issued from one asm block under one
// elect; step k's operands sit at fixed byte offsets from the tile bases (the
// descriptors' start-address field counts 16-byte units and cannot carry):
//   A (Q, two 64-d halves of 128 rows x 128 B): (k >> 2) * 16384 + (k & 3) * 32
//   B (K, two halves of 64 keys x 128 B):       (k >> 2) * 8192  + (k & 3) * 32
__device__ __forceinline__ void umma_s8_w(uint32_t tmem_d, uint64_t a0, uint64_t b0, uint32_t id) {
  asm volatile(
      "{\n.reg .pred e;\n.reg .b64 a<8>, b<8>;\n"
      "mov.b64 a0, %1;\nadd.s64 a1, %1, 2;\nadd.s64 a2, %1, 4;\nadd.s64 a3, %1, 6;\n"
      "add.s64 a4, %1, 1024;\nadd.s64 a5, %1, 1026;\nadd.s64 a6, %1, 1028;\nadd.s64 a7, %1, 1030;\n"
      "mov.b64 b0, %2;\nadd.s64 b1, %2, 2;\nadd.s64 b2, %2, 4;\nadd.s64 b3, %2, 6;\n"
      "add.s64 b4, %2, 512;\nadd.s64 b5, %2, 514;\nadd.s64 b6, %2, 516;\nadd.s64 b7, %2, 518;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a0, b0, %3, 0;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a4, b4, %3, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a5, b5, %3, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a6, b6, %3, 1;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a7, b7, %3, 1;\n}\n" ::"r"(tmem_d),
      "l"(a0), "l"(b0), "r"(id)
      : "memory");
}
// O += P.V of one key tile: up to four 16-key chunks j < nch, A = P chunk j in TMEM
// (8 columns from a_tmem), B = V chunk j (MN-major, 2048 B apart); the first step
// accumulates iff acc0
__device__ __forceinline__ void umma_pv4_w(uint32_t tmem_d, uint32_t a_tmem, uint64_t b0, uint32_t id, int nch,
                                           uint32_t acc0) {
  asm volatile(
      "{\n.reg .pred e, p0, p1, p2, p3, q0, pa;\n.reg .b64 b<4>;\n.reg .b32 t<4>;\n"
      "mov.b64 b0, %2;\nadd.s64 b1, %2, 128;\nadd.s64 b2, %2, 256;\nadd.s64 b3, %2, 384;\n"
      "mov.b32 t0, %1;\nadd.s32 t1, %1, 8;\nadd.s32 t2, %1, 16;\nadd.s32 t3, %1, 24;\n"
      "setp.ne.b32 pa, %5, 0;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "setp.gt.and.s32 p1, %4, 1, e;\nsetp.gt.and.s32 p2, %4, 2, e;\nsetp.gt.and.s32 p3, %4, 3, e;\n"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [t0], b0, %3, pa;\n"
      "@p1 tcgen05.mma.cta_group::1.kind::f16 [%0], [t1], b1, %3, 1;\n"
      "@p2 tcgen05.mma.cta_group::1.kind::f16 [%0], [t2], b2, %3, 1;\n"
      "@p3 tcgen05.mma.cta_group::1.kind::f16 [%0], [t3], b3, %3, 1;\n}\n" ::"r"(tmem_d),
      "r"(a_tmem), "l"(b0), "r"(id), "r"(nch), "r"(acc0)
      : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float *v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float *v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15]))
      : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t *w) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(w[0]),
               "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
               : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// packed two-lane FP32 (sm_100 FFMA2 / FADD2)
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n.reg .b64 ra, rb, rc, rd;\nmov.b64 ra, {%2, %3};\nmov.b64 rb, {%4, %5};\nmov.b64 rc, {%6, %7};\n"
      "fma.rn.f32x2 rd, ra, rb, rc;\nmov.b64 {%0, %1}, rd;\n}\n"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 d;
  asm("{\n.reg .b64 ra, rb, rd;\nmov.b64 ra, {%2, %3};\nmov.b64 rb, {%4, %5};\n"
      "add.rn.f32x2 rd, ra, rb;\nmov.b64 {%0, %1}, rd;\n}\n"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}

struct TcChunk {
  int lo, hi, tb, dir, blk, c;
};

// Lane-parallel chunk walk of the producers: a window of entries is loaded one per
// lane (two lanes per entry for 32-slot blocks), the entries' token offsets come
// from a warp prefix sum of the fill counts, the live chunks (live slot range,
// first token <= pos_max) are compacted into lanes 0 .. n-1 -- no per-chunk
// serial loop.  Same chunks, in the same logical order, as the serial walk of
// prefill_attention.cu (entries in logical order, P:711 live slot ranges).
struct PWalk {
  int wb, F, E, n, i;            // next entry to load, its first token; entries; window chunks, consumed
  int lo, hi, tb, dir, blk, c;   // this lane's compacted window chunk
};
__device__ __forceinline__ void pw_load(const PrefillParams &p, int r, int L, int pos_max, PWalk &w) {
  constexpr unsigned FULL = 0xffffffffu;
  const int lane = static_cast<int>(threadIdx.x & 31);
  const int cpe = p.bs >> 4, epw = 32 / cpe;   // chunks per entry (1 or 2), entries per window
  w.n = 0;
  w.i = 0;
  while (w.wb < w.E && w.F <= pos_max) {
    const int e = w.wb + lane / cpe, c = lane - (lane / cpe) * cpe;
    const bool in = lane < epw * cpe && e < w.E;
    int blk = 0, dir = 0, fill = 0;
    if (in) {
      blk = __ldg(p.bt + static_cast<int64_t>(r) * p.bt_stride + e);
      dir = __ldg(p.dirs + static_cast<int64_t>(r) * p.dir_rs + static_cast<int64_t>(e) * p.dir_cs);
      fill = p.fills ? static_cast<int>(__ldg(p.fills + static_cast<int64_t>(r) * p.fill_rs + e))
                     : min(p.bs, L - e * p.bs);
    }
    int incl = c == 0 ? fill : 0;   // inclusive prefix sum of the entries' fills
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += v;
    }
    const int Fe = w.F + incl - fill;   // first token of the entry
    const int lo_s = dir ? p.bs - fill : 0, hi_s = dir ? p.bs : fill;
    const int lo = max(lo_s - 16 * c, 0), hi = min(hi_s - 16 * c, 16);
    const int tb = dir ? Fe + p.bs - 1 - 16 * c : Fe + 16 * c;
    const int first = dir ? tb - (hi - 1) : tb + lo;
    const bool live = in && lo < hi && Fe <= pos_max && first <= pos_max;
    const unsigned mask = __ballot_sync(FULL, live);
    w.wb += epw;
    w.F += __shfl_sync(FULL, incl, 31);
    w.n = __popc(mask);
    const int src = lane < w.n ? static_cast<int>(__fns(mask, 0, lane + 1)) : 0;
    w.lo = __shfl_sync(FULL, lo, src);
    w.hi = __shfl_sync(FULL, hi, src);
    w.tb = __shfl_sync(FULL, tb, src);
    w.dir = __shfl_sync(FULL, dir, src);
    w.blk = __shfl_sync(FULL, blk, src);
    w.c = __shfl_sync(FULL, c, src);
    if (w.n > 0) return;
  }
}
// next key tile (up to kTcChunks chunks): lane j < count receives chunk j
__device__ __forceinline__ int pw_tile(const PrefillParams &p, int r, int L, int pos_max, PWalk &w, TcChunk &mine) {
  constexpr unsigned FULL = 0xffffffffu;
  const int lane = static_cast<int>(threadIdx.x & 31);
  int nch = 0;
#pragma unroll
  for (int j = 0; j < kTcChunks; ++j) {
    if (w.i == w.n) {
      pw_load(p, r, L, pos_max, w);
      if (w.n == 0) break;
    }
    const int i = w.i++;
    const int lo = __shfl_sync(FULL, w.lo, i), hi = __shfl_sync(FULL, w.hi, i), tb = __shfl_sync(FULL, w.tb, i);
    const int dir = __shfl_sync(FULL, w.dir, i), blk = __shfl_sync(FULL, w.blk, i), c = __shfl_sync(FULL, w.c, i);
    if (lane == j) mine = TcChunk{lo, hi, tb, dir, blk, c};
    ++nch;
  }
  return nch;
}

}  // namespace

// Dev-only cycle accounting (trace builds, -DBKV_DEV_TRACE): per CTA and role,
// cycles spent in each phase of the tile loop, read by bkv_dev_prefill_prof.
#ifdef BKV_DEV_TRACE
constexpr bool kTcProf = true;
#else
constexpr bool kTcProf = false;
#endif
constexpr int kProfSlots = 8;
__device__ unsigned long long g_tc_prof[148 * 3 * kProfSlots];
// event timeline of CTA 0 (trace builds): per warp, {clock64, tile << 16 | warp << 8 | event};
// each warp's lane 0 appends to its own region (no atomics on the traced path)
constexpr int kTraceWarps = 12, kTracePerWarp = 2048;
__device__ unsigned long long g_tc_trace[2 * kTraceWarps * kTracePerWarp];
__device__ unsigned int g_tc_tn[kTraceWarps];
__shared__ unsigned int s_tc_tn[kTraceWarps];   // per-warp event counts (shared: cheap to bump)
__device__ __forceinline__ void tc_event(int ev, int gt = 0) {
  if (kTcProf && blockIdx.x == 0 && (threadIdx.x & 31) == 0) {
    const int w = threadIdx.x >> 5;
    volatile unsigned int *cnt = s_tc_tn + w;
    const unsigned i = *cnt;
    if (i < kTracePerWarp) {
      unsigned long long *e = g_tc_trace + 2 * (w * kTracePerWarp + i);
      e[0] = clock64();
      e[1] = (static_cast<unsigned long long>(gt) << 16) | w << 8 | ev;
      *cnt = i + 1;
    }
  }
}

// QT = query tiles of 128 rows per CTA (1, or 2 "ping-pong" groups sharing every
// K/V tile: two softmax warpgroups, twice the MMA work per streamed byte).
template <int QT>
__global__ void __launch_bounds__(32 * (4 * QT + 3), 1)
    prefill_tc_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV,
                      const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmO,
                      const PrefillParams p) {
  constexpr int D = 128;
  constexpr int NS = QT == 1 ? kTcStages : 3;   // key-tile stages (shared memory budget)
  constexpr int MS = NS + 2;                     // tile metadata slots (one mbarrier each)
  constexpr int SMW = 4 * QT;                    // softmax warps
  constexpr int WK = SMW, WMMA = SMW + 1, WV = SMW + 2;   // K producer, MMA issuer, V producer
  constexpr int HALF = kTcKeys * 128;          // one 64-d half of a key tile: 64 rows x 128 B
  constexpr int TILE = 2 * HALF;               // K (or V) of one key tile
  constexpr int STAGE = 2 * TILE;              // K + V
  constexpr unsigned FULL = 0xffffffffu;

  extern __shared__ uint8_t smem_raw[];
  // a PDL-launched successor (the mixed dispatch's decode kernel, which reads
  // nothing this kernel writes) may take SMs as this grid's CTAs finish
  asm volatile("griddepcontrol.launch_dependents;");
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t *gb = smem_raw + (base - raw);
  const uint32_t sQ = base;                                  // QT x (2 halves x 128 rows x 128 B)
  const uint32_t sStage = sQ + QT * 2 * kTcRows * 128;       // NS key tiles (K | V)
  // output staging (o_tma): per query group, per softmax warp, per 64-d half: 32 rows x 128 B
  const uint32_t sO = sStage + NS * STAGE;
  const int n_ostage = p.o_tma ? QT : 0;
  // tile metadata ring (MS slots; see the producer): [slot][chunk], chunk count | last flag
  int4 *metas = reinterpret_cast<int4 *>(gb + (sO + n_ostage * 2 * kTcRows * 128 - base));
  int2 *tinfo = reinterpret_cast<int2 *>(metas + MS * kTcChunks);   // {chunks | flags, last token}
  // live requests (rows > 0) of batches up to kLiveCap, ascending: work items enumerate
  // these only, so a batch with many zero-row requests costs no empty-item search
  uint32_t *live_mask = reinterpret_cast<uint32_t *>(tinfo + MS);   // [kLiveCap / 32]
  uint16_t *live_list = reinterpret_cast<uint16_t *>(live_mask + kLiveCap / 32);
  int *live_n = reinterpret_cast<int *>(live_list + kLiveCap);
  uint64_t *bars = reinterpret_cast<uint64_t *>(live_n + 2);
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bars + 4 * NS + 8 * QT + 2 + MS);
  const uint32_t bar0 = smem_u32(bars);
  // K and V stages are handed over separately: a K stage frees as soon as the S
  // MMAs that read it complete (about two tiles before its V stage), so the K
  // stream runs further ahead of the MMA than a shared K|V ring allows
  const uint32_t fullK0 = bar0, fullV0 = bar0 + 8 * NS, emptyK0 = bar0 + 16 * NS, emptyV0 = bar0 + 24 * NS;
  // per query group q: s_full (S landed) and p_full/p_free (P written -- which
  // also frees the S buffer -- and P.V landed; p_free also marks "every P.V up
  // to this tile has landed in O"), two buffers each; q_full: Q staged
  const uint32_t grp0 = bar0 + 32 * NS;   // group q: + 64 q; s_full +0, (+16 unused), p_full +32, p_free +48
  const uint32_t q_full = grp0 + 64 * QT;
  const uint32_t q_free = q_full + 8;     // every S of the item's query tiles is done: Q may be replaced
  const uint32_t meta0 = q_free + 8;      // [MS]: tile metadata slot m published (all 32 K-producer lanes arrive)
  const bool q_tma = p.q_tma != 0;        // the K producer TMA-loads Q (else the softmax warps stage it)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  auto init_barriers = [&]() {
    for (int i = 0; i < NS; ++i) {
      mbar_init(fullK0 + 8 * i, 1);   // the K (V) producer arms its bytes
      mbar_init(fullV0 + 8 * i, 1);
      mbar_init(emptyK0 + 8 * i, 1);
      mbar_init(emptyV0 + 8 * i, 1);
    }
    for (int q = 0; q < QT; ++q)
      for (int b = 0; b < 2; ++b) {
        mbar_init(grp0 + 64 * q + 8 * b, 1);        // s_full
        mbar_init(grp0 + 64 * q + 32 + 8 * b, 4);   // p_full
        mbar_init(grp0 + 64 * q + 48 + 8 * b, 1);   // p_free
      }
    mbar_init(q_full, q_tma ? 1 : SMW);
    mbar_init(q_free, 1);
    for (int i = 0; i < MS; ++i) mbar_init(meta0 + 8 * i, 32);
    fence_mbar_init();
  };
  if (kTcProf && threadIdx.x < kTraceWarps) s_tc_tn[threadIdx.x] = 0;
  if (threadIdx.x == 0) {
    prefetch_tmap(&tmK);
    prefetch_tmap(&tmV);
    if (q_tma) prefetch_tmap(&tmQ);
    if (p.o_tma) prefetch_tmap(&tmO);
    init_barriers();
  }
  if (warp == WMMA) {   // TMEM per group q: S buffers at 256q + [0, 64) / [64, 128), O at 256q + [128, 256)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(256 * QT));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  const bool compact = p.B <= kLiveCap;
  constexpr int NW = 4 * QT + 3;
  if (compact) {   // one ballot mask per 32 requests
    for (int c = warp; c * 32 < p.B; c += NW) {
      const int r = c * 32 + lane;
      const bool live = r < p.B && __ldg(p.cu_q + r + 1) > __ldg(p.cu_q + r);
      const unsigned m = __ballot_sync(FULL, live);
      if (lane == 0) live_mask[c] = m;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (compact) {   // stable compaction: the same list in every CTA
    for (int c = warp; c * 32 < p.B; c += NW) {
      int off = 0;
      for (int k = 0; k < c; ++k) off += __popc(live_mask[k]);
      const unsigned m = live_mask[c];
      if ((m >> lane) & 1u) live_list[off + __popc(m & ((1u << lane) - 1u))] = static_cast<uint16_t>(c * 32 + lane);
      if (lane == 0 && (c + 1) * 32 >= p.B) *live_n = off + __popc(m);   // the last mask's warp
    }
    if (p.B == 0 && threadIdx.x == 0) *live_n = 0;
    __syncthreads();
  }
  const int nreq = compact ? *live_n : p.B;   // requests the work items enumerate
  auto req_of = [&](int i) -> int { return compact ? static_cast<int>(live_list[i]) : i; };

  // Persistent over work items (x, h, r), x = tile counted from the END of the
  // request (its latest, longest rows first): only existing tiles cost a pass;
  // no CTA is launched for an empty tile.  TMEM stays allocated and every
  // barrier keeps running phases across items: all roles number key tiles with
  // the same CTA-global counter gt (stage = gt % stages, S/P buffer = gt & 1),
  // so the producer already streams the next item while the current one drains.
  const int g = p.g;
  int gt0 = 0;           // key tiles of earlier items (identical in every role)
  int items_done = 0;
  const int n_items = ((p.tiles_max + QT - 1) / QT) * p.H * nreq;
  // First non-empty item >= from in this CTA's progression (from, from + G, ...):
  // the lanes of each warp test 32 candidates at once (warp-uniform result), so
  // the empty items of short or decode-only requests cost ~nothing.
  const int G = static_cast<int>(gridDim.x);
  auto next_item = [&](int from) -> int {
    const int HB = p.H * nreq;
    for (; from < n_items; from += 32 * G) {
      const int c = from + lane * G;
      bool live = false;
      if (c < n_items) {
        const int cx = c / HB, cr = req_of((c - cx * HB) / p.H);
        const int cn = __ldg(p.cu_q + cr + 1) - __ldg(p.cu_q + cr);
        live = (cn * g + kTcRows - 1) / kTcRows - 1 - QT * cx >= 0;
      }
      const unsigned m = __ballot_sync(FULL, live);
      if (m) return from + (__ffs(m) - 1) * G;
    }
    return n_items;
  };
  // item-level accounting (trace builds): role 2 slots 0 kernel cycles, 1 items,
  // 2 item start -> first tile metadata, 3 epilogue, 4 next-item search
  const long long k_t0 = kTcProf ? clock64() : 0;
  long long it_t = k_t0;
  auto iprof = [&](int slot, long long &t) {
    if (kTcProf && threadIdx.x == 0 && blockIdx.x < 148) {
      const long long c = clock64();
      atomicAdd(&g_tc_prof[(blockIdx.x * 3 + 2) * kProfSlots + slot], static_cast<unsigned long long>(c - t));
      t = c;
    }
  };
  for (int item = next_item(blockIdx.x); item < n_items; item = next_item(item + G)) {
  iprof(4, it_t);
  const int x = item / (p.H * nreq), hr = item - x * (p.H * nreq);
  const int ri = hr / p.H, h = hr - ri * p.H;
  const int r = req_of(ri);
  const int q0 = __ldg(p.cu_q + r);
  const int n = __ldg(p.cu_q + r + 1) - q0;
  const int rows = n * g;
  const int ntiles = (rows + kTcRows - 1) / kTcRows;
  const int tile_last = ntiles - 1 - QT * x;      // this item: tiles tile_last - QT + 1 .. tile_last
  if (tile_last < 0) continue;
  const int L = __ldg(p.seq_lens + r);
  // query tiles are aligned to the END of the request's rows: the latest rows fill
  // whole tiles, a partial tile holds the earliest rows (and its dead rows lie
  // before the request: the TMA Q box never reads past the request's last token)
  const int row_end = rows - QT * kTcRows * x;
  const int row0 = row_end - QT * kTcRows;   // may be negative: those rows (a whole group) are dead
  const int pos_max = L - n + (row_end - 1) / g;

  // Tile metadata: the producer walks the request's chunks (one tile of
  // lookahead, so each tile carries a "last" flag) and publishes per slot the
  // chunk count and (lo, hi, tb, dir) per chunk; every producer lane arrives on
  // the slot's mbarrier (release: each lane's own stores) and the MMA warp and
  // the softmax warps wait on its phase (acquire) -- independently: a named
  // barrier here made the eight softmax warps wait for the slowest every tile.
  // The tiles themselves are handed over by the stage mbarriers.

  long long ep_t = 0;
  if (warp == WK || warp == WV) {
    // ------------------------------------------------------------ producers
    // A key tile = up to four 16-slot chunks of the walk, each landing as rows
    // [16j, 16j+16) of the tile (one TMA box per 64-d half per tensor), so the
    // tile is one contiguous K-major (K) / MN-major (V) 128B-swizzled operand.
    // Warp 4 streams K and publishes the tile metadata (before its copies, so
    // the consumers can prepare), warp 6 streams V: 8 boxes per warp per tile.
    const bool is_k = warp == WK;
    tc_event(0);
    PWalk walk;
    walk.wb = 0;
    walk.F = 0;
    walk.E = p.fills ? __ldg(p.nent + r) : (L + p.bs - 1) / p.bs;
    walk.n = walk.i = 0;
    TcChunk ch{0, 0, 0, 0, 0, 0}, nx{0, 0, 0, 0, 0, 0};   // lane j: chunk j of the tile
    const uint64_t pol = policy_evict_last();   // every query tile of the request re-reads these
    int nch = pw_tile(p, r, L, pos_max, walk, ch);
    tc_event(1);
    if (is_k && q_tma) {
      // Q of the item's QT query tiles: one box {64 d, 1 half, g heads, 128/g tokens}
      // per 64-d half lands as 128 rows (token, head) x 128 B, 128B-swizzled -- the
      // K-major operand layout.  Rows before the request read earlier tokens (or
      // zero-fill below token 0); they are dead rows, masked by the softmax.  (The
      // whole warp waits: a lone spinning lane stalls the converged walk for long.)
      if (items_done > 0) mbar_wait(q_free, (items_done - 1) & 1);
      if (lane == 0) {
        mbar_arrive_expect_tx(q_full, QT * 2 * kTcRows * 128);
        const uint64_t pq = policy_evict_first();
#pragma unroll
        for (int q = 0; q < QT; ++q)
#pragma unroll
          for (int hf = 0; hf < 2; ++hf)
            tma_load_4d(sQ + q * (2 * kTcRows * 128) + hf * (kTcRows * 128), &tmQ, 0, hf, h * g,
                        q0 + (row0 + q * kTcRows) / g, q_full, pq);
      }
      __syncwarp();
    }
    if (is_k) tc_event(2);
    for (int t = 0; nch > 0; ++t) {
      const int nnx = pw_tile(p, r, L, pos_max, walk, nx);   // lookahead: is this tile the last?
      // metadata slot m of tile gt is rewritten for tile gt + MS only after K stage st
      // freed (S(gt + MS - NS) done), which follows p_full(gt + MS - NS - 2) = the
      // softmax finished that tile: with MS = NS + 2 every consumer has read slot m
      // (and waited on the phase of its mbarrier) by then
      const int gt = gt0 + t, st = gt % NS, round = gt / NS, m = gt % MS;
      if (round > 0) mbar_wait((is_k ? emptyK0 : emptyV0) + 8 * st, (round - 1) & 1);   // whole warp
      tc_event(3, gt);
      __syncwarp();
      if (is_k) {
        if (lane < nch) metas[m * kTcChunks + lane] = make_int4(ch.lo, ch.hi, ch.tb, ch.dir);
        // tile summary: the patch flag and the tile's largest live token (a row at
        // pos >= it with four whole chunks sees the whole tile: no masks)
        const bool part = lane < nch && (ch.lo > 0 || ch.hi < 16);
        const int last_tok = lane < nch ? (ch.dir ? ch.tb - ch.lo : ch.tb + ch.hi - 1) : -1;
        const unsigned pm = __ballot_sync(FULL, part);
        const int tmax = __reduce_max_sync(FULL, last_tok);
        if (lane == 0) tinfo[m] = make_int2(nch | (nnx == 0 ? kTcLastFlag : 0) | (pm ? kTcPatchFlag : 0), tmax);
        mbar_arrive(meta0 + 8 * m);   // (each lane: release of its own metadata stores)
      }
      const uint32_t fb = (is_k ? fullK0 : fullV0) + 8 * st;
      if (lane == 0) mbar_arrive_expect_tx(fb, nch * 2 * 2048);   // two 64-d half boxes per chunk
      __syncwarp();
      {   // lane 2j + hf copies half hf of chunk j
        const int j = (lane >> 1) & (kTcChunks - 1), hf = lane & 1;
        const int cj = __shfl_sync(FULL, ch.c, j), bj = __shfl_sync(FULL, ch.blk, j);
        const uint32_t dst = sStage + st * STAGE + (is_k ? 0 : TILE);
        if (lane < 2 * nch) tma_load_5d(dst + hf * HALF + j * 2048, is_k ? &tmK : &tmV, 0, 16 * cj, hf, h, bj, fb, pol);
      }
      __syncwarp();
      if (nnx == 0) {
        gt0 += t + 1;
        break;
      }
      nch = nnx;
      ch = nx;
    }
  } else if (warp == WMMA) {
    // ------------------------------------------------------------ MMA issuer
    // The whole warp walks the loop (waits, descriptors); one elected lane issues
    // each tcgen05.mma / commit (umma_w and friends).
    mbar_wait(q_full, items_done & 1);
    tc_fence_after();
    bool first_pv[QT];
#pragma unroll
    for (int q = 0; q < QT; ++q) first_pv[q] = true;
    auto issue_pv = [&](int gt, int nch) {   // P.V of key tile gt for every group, then free the V stage
      const int pb = gt & 1, st = gt % NS;
      const uint32_t idO = idesc(128, 128, 0, 1);
      mbar_wait(fullV0 + 8 * st, (gt / NS) & 1);   // V landed (and, patched, reached the softmax's p_full)
#pragma unroll
      for (int q = 0; q < QT; ++q) {
        mbar_wait(grp0 + 64 * q + 32 + 8 * pb, (gt >> 1) & 1);
        tc_event(17 + q, gt);
        tc_fence_after();
        // A = P of chunk j: 8 TMEM columns of the S buffer pb
        if (!(p.probe & 4)) umma_pv4_w(tmem + 256 * q + 128, tmem + 256 * q + pb * 64, sdesc(sStage + st * STAGE + TILE, HALF, 1024), idO,
                   nch, first_pv[q] ? 0u : 1u);
        first_pv[q] = false;
        umma_commit_w(grp0 + 64 * q + 48 + 8 * pb);
      }
      umma_commit_w(emptyV0 + 8 * st);
    };
    int prev_nch = 0;
    for (int t = 0;; ++t) {
      const int gt = gt0 + t, sb = gt & 1, st = gt % NS, m = gt % MS;
      long long pc0 = kTcProf ? clock64() : 0;
      auto prof = [&](int slot) {
        if (kTcProf && lane == 0 && blockIdx.x < 148) {
          const long long c = clock64();
          atomicAdd(&g_tc_prof[(blockIdx.x * 3 + 1) * kProfSlots + slot], static_cast<unsigned long long>(c - pc0));
          pc0 = c;
        }
      };
      mbar_wait(meta0 + 8 * m, (gt / MS) & 1);
      tc_event(10, gt);
      prof(0);
      const int tc = tinfo[m].x;
      const int nch = tc & 0xff;
      mbar_wait(fullK0 + 8 * st, (gt / NS) & 1);
      tc_event(11, gt);
      prof(1);
      const uint32_t idS = idesc(128, 16 * nch, 0, 0);
      const uint32_t sk = sStage + st * STAGE;
#pragma unroll
      for (int q = 0; q < QT; ++q) {
        // S(gt) reuses the S/P buffer of tile gt - 2: this thread already waited for that
        // tile's p_full (its P.V was issued in an earlier iteration), which each softmax
        // warp arrives after its last TMEM read of the buffer -- no separate s_free wait
        tc_event(15 + q, gt);
        tc_fence_after();
        static_assert(D == 128 && HALF == 8192 && kTcRows * 128 == 16384, "umma_s8_w operand offsets");
        if (!(p.probe & 2)) umma_s8_w(tmem + 256 * q + sb * 64, sdesc(sQ + q * (2 * kTcRows * 128), 16, 1024), sdesc(sk, 16, 1024), idS);
        umma_commit_w(grp0 + 64 * q + 8 * sb);
      }
      umma_commit_w(emptyK0 + 8 * st);               // K stage free once these S are done
      if (tc & kTcLastFlag) umma_commit_w(q_free);   // the item's last S: Q may be replaced
      tc_event(12, gt);
      prof(3);
      if (t >= 1) issue_pv(gt - 1, prev_nch);   // P.V of the previous tile overlaps S of this one
      tc_event(13, gt);
      prof(4);
      if (tc & kTcLastFlag) {
        issue_pv(gt, nch);
        tc_event(14, gt);
      }
      prev_nch = nch;
      if (tc & kTcLastFlag) {
        gt0 += t + 1;
        break;
      }
    }
  } else {
    // ------------------------------------------------------------ softmax warpgroup(s)
    const int qg = warp >> 2;                  // query group (128-row tile) of this warp
    const int row = (warp & 3) * 32 + lane;    // row of the group's tile = TMEM lane
    const int grow = row0 + qg * kTcRows + row;
    const bool ok = grow >= 0 && grow < row_end;
    const uint32_t s_full0 = grp0 + 64 * qg, p_full0 = s_full0 + 32,
                   p_free0 = s_full0 + 48;
    const uint32_t tq = tmem + 256 * qg;       // this group's TMEM columns
    const int tok = ok ? grow / g : 0, jh = ok ? grow - tok * g : 0;
    const int pos = ok ? L - n + tok : -1;
    if (!q_tma) {   // Q row -> shared memory (K-major, 128B swizzle, two 64-d halves)
      const uint4 *qs = reinterpret_cast<const uint4 *>(p.q + static_cast<int64_t>(q0 + tok) * p.q_st +
                                                        static_cast<int64_t>(h * g + jh) * p.q_sh);
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const uint4 v = ok ? __ldg(qs + c) : make_uint4(0u, 0u, 0u, 0u);
        st_shared_v4(sQ + qg * (2 * kTcRows * 128) + (c >> 3) * (kTcRows * 128) + tswz(row, c & 7), v);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(q_full);
    }
    const uint32_t lane_addr = static_cast<uint32_t>((warp & 3) * 32) << 16;
    float m_ref = -INFINITY, l = 0.f;
    int ntile = 0;
    for (;; ++ntile) {
      const int t = gt0 + ntile, sb = t & 1, st = t % NS, m = t % MS;   // CTA-global key tile number
      long long pc0 = kTcProf ? clock64() : 0;
      auto prof = [&](int slot) {
        if (kTcProf && threadIdx.x == 0 && blockIdx.x < 148) {
          const long long c = clock64();
          atomicAdd(&g_tc_prof[(blockIdx.x * 3 + 0) * kProfSlots + slot], static_cast<unsigned long long>(c - pc0));
          pc0 = c;
        }
      };
      if ((warp & 3) == 0) tc_event(20, t);
      mbar_wait(meta0 + 8 * m, (t / MS) & 1);
      if ((warp & 3) == 0) tc_event(21, t);
      if (ntile == 0) iprof(2, it_t);
      prof(0);
      const int2 ti = tinfo[m];
      const int tc = ti.x;
      const int nch = tc & 0xff;
      auto load_meta = [&](int4 (&meta)[kTcChunks]) {
#pragma unroll
        for (int j = 0; j < kTcChunks; ++j) meta[j] = j < nch ? metas[m * kTcChunks + j] : make_int4(0, 0, 0, 0);
      };
      // dead V rows of partly live chunks -> zero (P = 0 must never meet NaN, reading Q10);
      // only then does the softmax wait for the tile's copies itself (S implies K landed)
      if (qg == 0 && (tc & kTcPatchFlag)) {   // group 0 patches for all
        int4 meta[kTcChunks];
        load_meta(meta);
        mbar_wait(fullV0 + 8 * st, (t / NS) & 1);   // the tile's V landed
#pragma unroll
        for (int j = 0; j < kTcChunks; ++j) {   // unrolled: meta[] stays in registers
          if (j < nch && (meta[j].x > 0 || meta[j].y < 16)) {
            const uint32_t sv = sStage + st * STAGE + TILE + j * 2048;
#pragma unroll
            for (int q = 0; q < 256; q += kTcRows) {   // 16 slots x 2 halves x 8 pieces
              const int slot = (q + row) >> 4, rest = (q + row) & 15;
              if (slot < meta[j].x || slot >= meta[j].y) sts128_zero(sv + (rest >> 3) * HALF + slot * 128 + (rest & 7) * 16);
            }
          }
        }
      }
      prof(1);
      // S tile -> registers
      prof(2);
      mbar_wait(s_full0 + 8 * sb, (t >> 1) & 1);
      tc_event(22, t);
      prof(3);
      tc_fence_after();
      float s[kTcChunks * 16];
#pragma unroll
      for (int j = 0; j < kTcChunks; ++j)   // (columns of chunks >= nch: stale, masked below)
        tmem_ld16(tq + lane_addr + sb * 64 + 16 * j, s + 16 * j);
      tmem_wait_ld();
      // per chunk, the live slots of this row form one interval [clo, chi): the
      // entry's live range intersected with the causal bound (forward: token
      // tb + c <= pos -> c <= pos - tb; reversed: tb - c <= pos -> c >= tb - pos)
      // With a positive scale the max commutes with the scaling, which is then
      // folded into the exponent (p = 2^(s*scale - m)); a tile every row of the
      // warp sees whole (four full chunks before its first query) skips the masks.
      const bool fold = p.scale_log2 > 0.f;
      const bool whole = nch == kTcChunks && !(tc & kTcPatchFlag) && pos >= ti.y;
      // masks (unless every row of the warp sees the whole tile): dead slots -> -inf;
      // without the fold the scores are scaled here
      if (!(fold && __all_sync(FULL, whole))) {
        int4 meta[kTcChunks];
        load_meta(meta);
        int clo[kTcChunks], chi[kTcChunks];
#pragma unroll
        for (int j = 0; j < kTcChunks; ++j) {
          clo[j] = meta[j].x;
          chi[j] = meta[j].y;
          if (meta[j].w) clo[j] = max(clo[j], meta[j].z - pos);
          else chi[j] = min(chi[j], pos - meta[j].z + 1);
          if (j >= nch) chi[j] = 0;
        }
#pragma unroll
        for (int j = 0; j < kTcChunks; ++j) {
#pragma unroll
          for (int c = 0; c < 16; ++c) {
            const float v = fold ? s[16 * j + c] : s[16 * j + c] * p.scale_log2;
            s[16 * j + c] = (c >= clo[j] && c < chi[j]) ? v : -INFINITY;
          }
        }
      }
      // P = 2^(s * scale - base) into TMEM over the S buffer sb just read (bf16 pairs,
      // columns 8j .. 8j + 7 per 16-key chunk), branch-free over the four chunks
      // (chunks >= nch hold -inf: p = 0, in P columns no P.V reads); scale-and-shift
      // and the row sums on the packed two-lane FP32 pipe (FFMA2 / FADD2).  Returns
      // the row sum; xmax = the largest exponent.  S(t + 2) reuses the buffer: it is
      // issued after p_full below and after P.V(t) (one thread's MMAs run in order).
      auto exp_store = [&](float base, float &xmax) -> float {
        const float2 sc = make_float2(p.scale_log2, p.scale_log2), nb = make_float2(-base, -base);
        float2 l2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        float xm[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int j = 0; j < kTcChunks; ++j) {
          uint32_t pw[8];
#pragma unroll
          for (int c = 0; c < 16; c += 2) {
            const float2 x = ffma2(make_float2(s[16 * j + c], s[16 * j + c + 1]), sc, nb);
            xm[(c >> 1) & 3] = fmaxf(xm[(c >> 1) & 3], fmaxf(x.x, x.y));
            const float p0 = ex2(x.x), p1 = ex2(x.y);
            l2[(c >> 1) & 1] = fadd2(l2[(c >> 1) & 1], make_float2(p0, p1));
            pw[c >> 1] = pack_bf16(p0, p1);
          }
          tmem_st8(tq + lane_addr + sb * 64 + 8 * j, pw);
        }
        xmax = fmaxf(fmaxf(xm[0], xm[1]), fmaxf(xm[2], xm[3]));
        return (l2[0].x + l2[1].x) + (l2[0].y + l2[1].y);
      };
      // Speculative pass: exponentiate against the running reference straight away
      // (no max -> exponent dependency); it stands unless a row has no reference yet or
      // a live score passes it by more than 8 (p > 2^8) -- then the exact pass below
      // (row max, lazy rescale) recomputes and overwrites P.  Warp-uniform decision.
      bool redo = true;
      if (p.probe & 1) {   // dev what-if: no exponentials (P = 0 stored)
        const uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
        for (int j = 0; j < kTcChunks; ++j) tmem_st8(tq + lane_addr + sb * 64 + 8 * j, z);
        redo = false;
      } else if (fold && ntile > 0) {   // (an item's first tile has no reference yet)
        float xmax;
        const float ls = exp_store(m_ref, xmax);
        redo = __any_sync(FULL, !(m_ref > -INFINITY) || xmax > 8.f);
        if (!redo) l += ls;
      }
      if (redo) {
      if (fold) tmem_wait_st();   // the speculative P stores land before their overwrite
      // eight independent max chains (a single running max is a 64-deep
      // dependency chain on one thread)
      float mx8[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mx8[i] = -INFINITY;
#pragma unroll
      for (int c = 0; c < kTcChunks * 16; ++c) mx8[c & 7] = fmaxf(mx8[c & 7], s[c]);
      float mx = fmaxf(fmaxf(fmaxf(mx8[0], mx8[1]), fmaxf(mx8[2], mx8[3])),
                       fmaxf(fmaxf(mx8[4], mx8[5]), fmaxf(mx8[6], mx8[7])));
      if (fold) mx *= p.scale_log2;   // (-inf stays -inf)
      // lazy rescale: the reference max moves only when it grows by more than 8
      // (2^8 headroom for p); O in TMEM is rescaled warp-collectively, and only
      // once every earlier P.V has landed (p_free of the previous tile)
      const bool grow = mx > m_ref + 8.f;
      const bool resc = grow && m_ref != -INFINITY;
      if (__any_sync(FULL, resc)) {
        const float alpha = resc ? ex2(m_ref - mx) : 1.f;
        l *= alpha;
        mbar_wait(p_free0 + 8 * ((t - 1) & 1), ((t - 1) >> 1) & 1);   // (t >= 1: m_ref set by an earlier tile)
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < D; c += 16) {
          float o[16];
          tmem_ld16(tq + lane_addr + 128 + c, o);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; ++i) o[i] *= alpha;
          tmem_st16(tq + lane_addr + 128 + c, o);
        }
        tmem_wait_st();
        tc_fence_before();
      }
      if (grow) m_ref = mx;
      const float base_m = m_ref == -INFINITY ? 0.f : m_ref;
      if (fold) {
        float xmax;
        l += exp_store(base_m, xmax);
      } else {
      float l4[4] = {0.f, 0.f, 0.f, 0.f};   // independent row-sum chains, folded into l below
#pragma unroll
      for (int j = 0; j < kTcChunks; ++j) {
        if (j >= nch) break;
        uint32_t pw[8];
#pragma unroll
        for (int c = 0; c < 16; c += 2) {
          const float x0 = fold ? fmaf(s[16 * j + c], p.scale_log2, -base_m) : s[16 * j + c] - base_m;
          const float x1 = fold ? fmaf(s[16 * j + c + 1], p.scale_log2, -base_m) : s[16 * j + c + 1] - base_m;
          const float p0 = ex2(x0), p1 = ex2(x1);
          l4[(c >> 1) & 3] += p0 + p1;
          pw[c >> 1] = pack_bf16(p0, p1);
        }
        tmem_st8(tq + lane_addr + sb * 64 + 8 * j, pw);
      }
      l += (l4[0] + l4[1]) + (l4[2] + l4[3]);
      }
      }   // redo
      tmem_wait_st();
      if (qg == 0 && (tc & kTcPatchFlag)) fence_proxy_async_smem();   // zeroed V rows: generic writes the MMA reads
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full0 + 8 * sb);   // (also frees the S buffer for S(t + 2))
      tc_event(23, t);
      prof(6);
      if (kTcProf && threadIdx.x == 0 && blockIdx.x < 148) atomicAdd(&g_tc_prof[(blockIdx.x * 3 + 0) * kProfSlots + 7], 1ull);
      if (tc & kTcLastFlag) {
        ++ntile;
        break;
      }
    }
    // ---- epilogue: O / l -> bf16 rows, once the last P.V landed
    if (kTcProf) ep_t = clock64();
    if ((warp & 3) == 0) tc_event(24);
    gt0 += ntile;
    mbar_wait(p_free0 + 8 * ((gt0 - 1) & 1), ((gt0 - 1) >> 1) & 1);
    tc_fence_after();
    if ((warp & 3) == 0) tc_event(25);
    const float inv = l > 0.f ? 1.f / l : 0.f;
    // whole warps of live rows stage their 32 rows in shared memory (128B-swizzled,
    // conflict-free) and one lane TMA-stores them: coalesced 128-byte lines instead
    // of 32 row-strided 16-byte stores per instruction.  Warps with dead rows (a
    // request's first item) store their live rows directly.
    const bool o_tma = p.o_tma && __all_sync(FULL, ok);
    const uint32_t so = sO + qg * (2 * kTcRows * 128) + (warp & 3) * (2 * 32 * 128);   // [half][32 rows][128 B]
    if (o_tma) {
      if (lane == 0) bulk_wait_read_all();   // this warp's previous store has left the staging buffer
      __syncwarp();
    }
    uint4 *orow = reinterpret_cast<uint4 *>(p.out + static_cast<int64_t>(q0 + tok) * p.o_st +
                                            static_cast<int64_t>(h * g + jh) * p.o_sh);
    auto put32 = [&](const float (&o)[32], int c0) {   // 32 columns -> bf16 -> staging / row
#pragma unroll
      for (int c = 0; c < 32; c += 8) {
        const uint4 w = make_uint4(pack_bf16(o[c] * inv, o[c + 1] * inv), pack_bf16(o[c + 2] * inv, o[c + 3] * inv),
                                   pack_bf16(o[c + 4] * inv, o[c + 5] * inv), pack_bf16(o[c + 6] * inv, o[c + 7] * inv));
        const int k = (c0 + c) / 8;   // 16-byte chunk of the row: half k / 8, chunk k % 8
        if (o_tma) st_shared_v4(so + (k >> 3) * (32 * 128) + tswz(lane, k & 7), w);
        else if (ok) orow[k] = w;
      }
    };
    // 32 columns per TMEM load, the next batch in flight while this one is packed
    float oa[32], ob[32];
    tmem_ld16(tq + lane_addr + 128, oa);
    tmem_ld16(tq + lane_addr + 144, oa + 16);
    tmem_wait_ld();
#pragma unroll
    for (int c0 = 0; c0 < D; c0 += 64) {
      tmem_ld16(tq + lane_addr + 128 + c0 + 32, ob);
      tmem_ld16(tq + lane_addr + 128 + c0 + 48, ob + 16);
      put32(oa, c0);
      tmem_wait_ld();
      if (c0 + 64 < D) {
        tmem_ld16(tq + lane_addr + 128 + c0 + 64, oa);
        tmem_ld16(tq + lane_addr + 128 + c0 + 80, oa + 16);
      }
      put32(ob, c0 + 32);
      if (c0 + 64 < D) tmem_wait_ld();
    }
    if (o_tma) {
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        const int tok0 = q0 + (row0 + qg * kTcRows + (warp & 3) * 32) / g;
        tma_store_4d(&tmO, so, 0, 0, h * g, tok0);
        tma_store_4d(&tmO, so + 32 * 128, 0, 1, h * g, tok0);
        bulk_commit();
      }
    }
    tc_fence_before();
  }
  if (warp < SMW) {
    if ((warp & 3) == 0) tc_event(26);
    iprof(3, ep_t);
    if (kTcProf && threadIdx.x == 0 && blockIdx.x < 148) atomicAdd(&g_tc_prof[(blockIdx.x * 3 + 2) * kProfSlots + 1], 1ull);
    it_t = kTcProf ? clock64() : 0;
  }
  ++items_done;
  }   // work items
  {
    long long t0 = k_t0;
    iprof(0, t0);
  }
  if (p.o_tma && warp < SMW && lane == 0) bulk_wait_all();   // staged output stores complete
  __syncthreads();
  if (warp == WMMA) {   // the allocating warp frees the TMEM columns
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256 * QT));
  }
}

}  // namespace bkv

extern "C" __attribute__((visibility("default"))) int bkv_dev_prefill_trace(unsigned long long *host, int reset) {
  cudaError_t e = cudaMemcpyFromSymbol(host, bkv::g_tc_trace, sizeof(bkv::g_tc_trace));
  if (reset) {
    static unsigned z[bkv::kTraceWarps] = {};
    static unsigned long long zz[2 * bkv::kTraceWarps * bkv::kTracePerWarp] = {};
    cudaMemcpyToSymbol(bkv::g_tc_tn, z, sizeof(z));
    cudaMemcpyToSymbol(bkv::g_tc_trace, zz, sizeof(zz));
  }
  return e == cudaSuccess ? bkv::kTraceWarps * bkv::kTracePerWarp : -1;
}

extern "C" __attribute__((visibility("default"))) int bkv_dev_prefill_prof(unsigned long long *host, int reset) {
  cudaError_t e = cudaMemcpyFromSymbol(host, bkv::g_tc_prof, sizeof(bkv::g_tc_prof));
  if (reset) {
    static unsigned long long zeros[148 * 3 * bkv::kProfSlots] = {};
    cudaMemcpyToSymbol(bkv::g_tc_prof, zeros, sizeof(zeros));
  }
  return e == cudaSuccess ? (bkv::kTcProf ? 1 : 2) : -1;
}

namespace bkv {

template <int QT>
static int tc_smem_bytes(bool o_tma) {
  constexpr int NS = QT == 1 ? kTcStages : 3;
  constexpr int MS = NS + 2;
  return 1024 + QT * 2 * kTcRows * 128 * (o_tma ? 2 : 1) + NS * 4 * kTcKeys * 128 +
         MS * kTcChunks * 16 + MS * 8 + kLiveCap / 32 * 4 + kLiveCap * 2 + 8 + (4 * NS + 8 * QT + 2 + MS) * 8 + 16;   // + metadata, barriers, TMEM slot
}

int prefill_tc_smem_bytes() { return tc_smem_bytes<1>(false); }

template <int QT>
static cudaError_t launch_tc(const CUtensorMap &tmK, const CUtensorMap &tmV, const CUtensorMap *tmQ,
                             const CUtensorMap *tmO, const PrefillParams &p, int max_q_len, cudaStream_t s) {
  const int smem = tc_smem_bytes<QT>(tmO != nullptr);
  {
    cudaError_t e = ensure_dyn_smem(reinterpret_cast<const void *>(prefill_tc_kernel<QT>), smem);
    if (e != cudaSuccess) return e;
  }
  const long long tiles = (static_cast<long long>(max_q_len) * p.g + kTcRows - 1) / kTcRows;
  PrefillParams q = p;
  q.tiles_max = static_cast<int>(tiles);
  q.q_tma = tmQ != nullptr;
  q.o_tma = tmO != nullptr;
  DevProps dp;
  {
    cudaError_t e = dev_props(&dp);
    if (e != cudaSuccess) return e;
  }
  const int sms = dp.sms;
  const long long items = ((tiles + QT - 1) / QT) * p.H * p.B;
  const int cap = p.sm_reserve > 0 && p.sm_reserve < sms ? sms - p.sm_reserve : sms;
  const int grid = static_cast<int>(items < cap ? items : cap);   // one persistent CTA per SM
  prefill_tc_kernel<QT><<<grid, 32 * (4 * QT + 3), smem, s>>>(tmK, tmV, tmQ ? *tmQ : tmK, tmO ? *tmO : tmK, q);
  return cudaGetLastError();
}

cudaError_t launch_prefill_tc(const CUtensorMap &tmK, const CUtensorMap &tmV, const CUtensorMap *tmQ,
                              const CUtensorMap *tmO, const PrefillParams &p, int max_q_len, cudaStream_t s) {
  // default: two ping-pong 128-row query tiles per CTA share every K/V tile (Llama-70B
  // TP1 prefill rows 191 -> 233 TF/s); BKV_PREFILL_QT=1 (dev) runs one tile per CTA
  if (dev_switches().prefill_qt == 1) return launch_tc<1>(tmK, tmV, tmQ, tmO, p, max_q_len, s);
  return launch_tc<2>(tmK, tmV, tmQ, tmO, p, max_q_len, s);
}

}  // namespace bkv
