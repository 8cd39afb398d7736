// bkv_internal.h -- declarations shared by the bkv translation units (not part
// of the public ABI; include/bkv.h is).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace bkv {

// ---------------------------------------------------------------- kv_append
struct AppendParams {
  uint16_t *k, *v;  // pool (bf16 bits)
  int64_t sb, sh, ss;
  int H, bs;
  const int32_t *bt;
  int bt_stride;
  const uint8_t *dirs;
  int dir_rs, dir_cs;
  const int32_t *before;
  const int32_t *cu_new;
  const uint16_t *k_new, *v_new;
  int64_t *slot_mapping;  // optional
  int B;
  // general map: per-entry fill counts; nullptr for a dense map
  const uint8_t *fills;
  int fill_rs;
  const int32_t *nent;
  int max_entries;        // bt_stride: sizes the per-CTA prefix table in shared memory
  // fused lazy checkpoint: evict[i] >= 0 -> the old rows of new
  // token i's slot go to row evict[i] of ck_k / ck_v before the overwrite
  const int32_t *evict;
  uint16_t *ck_k, *ck_v;
};
cudaError_t launch_kv_append(const AppendParams &p, int head_dim, cudaStream_t s);

// lazy-checkpoint gather / restore scatter of whole slots (all heads, K and V)
struct SlotCopyParams {
  uint16_t *k, *v;  // pool
  int64_t sb, sh, ss;
  int H, bs;
  const int64_t *slots;
  int n;
  uint16_t *buf_k, *buf_v;  // [n][H][d] contiguous
  int restore;              // 0: pool -> buf (checkpoint), 1: buf -> pool (restore)
};
cudaError_t launch_slot_copy(const SlotCopyParams &p, int head_dim, cudaStream_t s);

// ------------------------------------------------------- decode attention
struct DecodeParams {
  const int32_t *bt;
  int bt_stride;
  const uint8_t *dirs;
  int dir_rs, dir_cs;
  const int32_t *seq_lens;
  const uint8_t *fills;  // general map (f3): entry fill counts, nullptr for a dense map
  int fill_rs;
  const int32_t *nent;   // general map: entries per request
  int B, H, bs, g;
  const uint16_t *q;
  int64_t q_ss, q_sh;
  uint16_t *out;
  int64_t o_ss, o_sh;
  float scale_log2;      // softmax_scale * log2(e)
  int *sched;            // [0] next unit, [1] exited CTAs (re-armed to 0 by the merge kernel or the last CTA)
  int *merge_cnt;        // [B*H] split arrivals per (request, kv head) for the fused merge (self-cleaning)
  int fused_merge;       // 1: last-arriver merge inside the decode kernel (no merge kernel launch)
  int kv_mode;           // 0: separate K and V boxes; 1/2: one K|V box (tmK = combined map), K resp. V first
  int *plan_out;         // split plan published by CTA 0 for the merge kernel
  float *part_ml;        // [units_max][g][2]  (m in log2 domain, l)
  float *part_o;         // [units_max][g][D]  un-normalised partial outputs
  int target_units;      // split plan: aim for about this many units
  int min_split;         // split plan: at least this many blocks per unit (large problems)
  int small_plan;        // split plan: chain-balanced P for small problems (BKV_SMALL_PLAN=0: off)
  int streamk;           // small problems: equal contiguous block ranges per warp (rows cut across warps)
  int units_max;         // workspace capacity in units
  int slots;             // ring depth per warp (S)
  int q_bytes;           // smem bytes per q-ring entry
  int total_warps;       // grid * warps per CTA
  int pdl;               // launched with programmatic dependent launch (BKV_FLAG_PDL)
  int pdl_nowait;        // PDL, and the preceding kernel is independent (mixed dispatch): skip the grid wait
  // fused decode step (bkv_decode_step): new token rows [B][H][D] + pool for the write; k_new == nullptr otherwise
  const uint16_t *k_new, *v_new;
  uint16_t *k_pool, *v_pool;
  int64_t pool_sb, pool_sh, pool_ss;
  // fused reassembly (f2): the merge kernel also stores every output row into
  // these device-accessible outputs (peers' buffers over NVLink), same strides
  uint16_t *peer_out[8];
  int n_peers;
  int peer_mc;   // peer_out[0] is an NVLS multicast address (one multimem store reaches every rank)
  int debug_flags;       // dev only: 1 = skip the math (data-movement skeleton), 2 = merge re-arm only, 4 = CTA-major first units, 8 = exit after the plan, 16 = exit at entry, 32 = no early PDL trigger
  unsigned long long *trace;  // dev only (BKV_TRACE): per-warp event log, else nullptr
  int trace_cap;         // events per warp
};

struct DecodeLaunch {
  int grid, warps, smem_bytes;
};

// Grid / ring configuration for (head_dim, group) on the current device.
cudaError_t decode_config(int head_dim, int group, int num_seqs, DecodeLaunch *cfg,
                          int *slots, int *q_bytes);
int decode_target_units(const DecodeLaunch &cfg);
int decode_min_split(int group);
cudaError_t launch_decode(const CUtensorMap &tmK, const CUtensorMap &tmV, const DecodeParams &p,
                          int head_dim, const DecodeLaunch &cfg, cudaStream_t s);

// ------------------------------------------- mixed prefill + decode (f4)
struct PrefillParams {
  const int32_t *bt;
  int bt_stride;
  const uint8_t *dirs;
  int dir_rs, dir_cs;
  const uint8_t *fills;   // general map (f3) or nullptr
  int fill_rs;
  const int32_t *nent;
  const int32_t *seq_lens;
  const int32_t *cu_q;    // [B+1] query rows of request r: its last cu_q[r+1]-cu_q[r] tokens
  int B, H, bs, g;
  const uint16_t *q;
  int64_t q_st, q_sh;
  uint16_t *out;
  int64_t o_st, o_sh;
  float scale_log2;
  int tiles_max;          // 128-row query tiles of the longest request (persistent kernels)
  int q_tma;              // tcgen05 kernel: Q tiles arrive by TMA (tmQ; needs g | 128)
  int sm_reserve;         // tcgen05 kernel: SMs its persistent grid leaves free (mixed dispatch)
  int o_tma;              // tcgen05 kernel: whole-warp output rows leave by TMA store (tmO; g | 32)
  int probe;              // dev what-if timing probes (BKV_PREFILL_PROBE, only in builds with
                          // -DBKV_DEV_PROBES or the trace build; results are wrong): 1 no exp,
                          // 2 no S MMAs, 4 no P.V MMAs
};
int prefill_smem_bytes(int head_dim);
bool prefill_uses_tc(int head_dim);   // tcgen05 kernel (wants 1-half TMA boxes)
cudaError_t launch_prefill(const CUtensorMap &tmK, const CUtensorMap &tmV, const CUtensorMap *tmQ,
                           const CUtensorMap *tmO, const PrefillParams &p, int head_dim, int max_q_len, cudaStream_t s);
cudaError_t launch_prefill_tc(const CUtensorMap &tmK, const CUtensorMap &tmV, const CUtensorMap *tmQ,
                              const CUtensorMap *tmO, const PrefillParams &p, int max_q_len, cudaStream_t s);

// cross-rank completion signal of the fused reassembly (f2)
struct PeerBarrierParams {
  uint32_t *pads[8];     // pads[k] = peer k's flag array (device-accessible), [n] entries
  int n, rank;
  uint32_t *counter;     // this rank's epoch counter (device)
  uint32_t *err;         // set to 1 on timeout
  unsigned long long timeout_ns;
};
cudaError_t launch_peer_barrier(const PeerBarrierParams &p, cudaStream_t s);
constexpr int kMaxPeers = 8;

// ------------------------------------ planned decode (static split plan)
// A decode plan is built on the HOST once per step from the scheduler's host
// seq_lens (bkv_decode_plan, csrc/decode_plan.cu) and reused by every layer's
// bkv_decode_planned call ("computed on device or host").
// Buffer = int32 words: PlanHeader, then the arrays at the header's offsets.
constexpr int32_t kPlanMagic = 0x504b5642;   // "BVKP"
constexpr int32_t kPlanVersion = 1;
constexpr int kPlanSplitBit = 30;            // seg.w = e1 | split << 30
struct PlanHeader {
  int32_t magic, version, words;             // words = total int32 words of the plan
  int32_t B, H, g, D, bs, general;           // geometry the plan was built for
  int32_t grid, warps;                       // launch it was built for (grid = SMs, one CTA each)
  int32_t P;                                 // blocks per warp range
  int32_t n_segs, n_tasks, n_zero;
  int32_t total;                             // N = sum_r nb_r * H (blocks x kv heads)
  int32_t off_wseg;                          // int32 [grid*warps + 1]: segments of warp w
  int32_t off_segs;                          // 2 x int4 [n_segs] {r, h, e0, e1 | split << 30}, {L, nb, 0, 0}
  int32_t off_ctask;                         // int32 [grid + 1]: merge tasks of CTA c
  int32_t off_tasks;                         // int4  [2 * n_tasks] (see PlanTask)
  int32_t off_zero;                          // int32 [2 * n_zero] {r, h}: rows with no tokens
  int32_t max_pieces;                        // largest n of a cross-CTA row
  int32_t max_entries;                       // bt_stride the plan was checked against
  int32_t off_xrows, n_xrows;                // int4 [n_xrows] {r, h, c0, n | flag0 << 16}: rows cut across CTAs
  int32_t off_ent, n_ent;                    // uint32 [total]: the step's entries in flattened (r, h, e) order
  int32_t reserved[5];
};
// packed flattened entry: block id | direction << 25 | (live tokens - 1) << 26 | last entry of the row << 31
constexpr uint32_t kEntBlockMask = (1u << 25) - 1;
constexpr int kEntDirShift = 25, kEntFillShift = 26, kEntLastShift = 31;
static_assert(sizeof(PlanHeader) == 32 * 4, "plan header is 32 words");
// A merge task (two int4) combines the pieces of one (request r, kv head h) row
// that lie in warps wa..wb of one CTA (piece k in warp wa+k: shared-memory slot
// wa_slot for k = 0, slot 0 otherwise).  mode 0: the row lies in this CTA only
// -> bf16 output.  mode 1: the row crosses CTAs c0 .. c0+n-1; this CTA's
// combined piece goes to global slot gslot and the last CTA to arrive merges
// the n pieces in CTA order (global slot of piece k: k ? 2(c0+k) : 2 c0 + flag0).
struct PlanTask {
  int32_t r, h, warps, mode;   // warps = wa | wb << 8 | wa_slot << 16 (CTA-local warp ids)
  int32_t c0, n, flag0, gslot;
};
size_t plan_words_bound(int B, int H, int bt_stride, int grid, int warps);
struct HostMap {   // the host copy of a step's block map (bkv_block_map with host pointers)
  const int32_t *bt;
  int bt_stride;
  const uint8_t *dirs;
  int dir_rs, dir_cs;
  const uint8_t *fills;   // general map or nullptr
  int fill_rs;
  const int32_t *nent;
};
const char *build_plan(const int32_t *seq_lens, const HostMap &map, int B, int H, int g, int D, int bs, int grid,
                       int warps, int32_t *out, size_t out_words, size_t *used_words);
constexpr int kPlannedWarps = 8;             // warps per CTA of the planned kernel

struct __align__(16) PlannedParams {
  const int32_t *bt;
  int bt_stride;
  const uint8_t *dirs;
  int dir_rs, dir_cs;
  const int32_t *seq_lens;
  const uint8_t *fills;  // general map (f3) or nullptr
  int fill_rs;
  const int32_t *nent;
  int B, H, bs, g;
  const uint16_t *q;
  int64_t q_ss, q_sh;
  uint16_t *out;
  int64_t o_ss, o_sh;
  float scale_log2;
  // the plan (device copy of the host-built buffer)
  const int32_t *wseg;   // [W + 1]
  const int4 *segs;      // 2 per segment: {r, h, e0, e1 | split << 30}, {L_r, entries of r, 0, 0}
  const int32_t *ctask;  // [grid + 1]
  const int4 *tasks;     // 2 per task (PlanTask)
  const int32_t *zero;   // {r, h} pairs
  const int4 *xrows;     // rows cut across CTAs (merged by planned_xmerge_kernel)
  const int32_t *plan_hdr;   // device copy of the PlanHeader: per-step values (P, n_zero, n_xrows)
  const uint32_t *ent;       // packed flattened entries (block, dir, fill, last) in warp order
  int xrows_cap;         // capacity of xrows (sizes the merge kernel's grid; graph-safe)
  float *gpiece;         // [2*grid][g*(D+2)] cross-CTA pieces
  int slots, pdl, kv_mode;
  int kv_early;          // BKV_FLAG_KV_EARLY: first ring tiles requested before the PDL grid wait
  int pf;                // kv_early: the warp's first pf entries are also prefetched into L2 before the wait
  const uint16_t *k_new, *v_new;   // fused decode step (f2), nullptr otherwise
  uint16_t *k_pool, *v_pool;
  int64_t pool_sb, pool_sh, pool_ss;
  uint16_t *peer_out[8];
  int n_peers;
  int peer_mc;   // peer_out[0] is an NVLS multicast address (one multimem store reaches every rank)
  unsigned long long *trace;   // dev only (trace build, BKV_TRACE >= 4): 8 %globaltimer stamps per warp
};
int planned_smem_bytes(int head_dim, int group, int slots, int warps);
int planned_piece_floats(int group, int head_dim);   // floats per cross-CTA piece slot
cudaError_t launch_planned(const CUtensorMap &tmK, const CUtensorMap &tmV, const PlannedParams &p,
                           int head_dim, int grid, int warps, int smem_bytes, cudaStream_t s);
// Developer switches (DESIGN.md §7 table), read from the environment ONCE per
// process and again only on bkv_reload_dev_switches().  BKV_DEBUG (probes that
// skip work) is honoured only by a BKV_DEV_TRACE build.
struct DevSwitches {
  int slots, warps, ctas_per_sm, units_per_warp, min_split /* -1: default */, small_plan, streamk;
  int merge_warps, fused_merge, kv_combined, mha_cuda_cores, prefill_mma_sync, prefill_qt, prefill_q_ldg, prefill_o_stg, prefill_probe, mixed_reserve;
  int mixed_overlap, debug, trace, planned_slots, planned_dynamic_p, planned_pf;
};
const DevSwitches &dev_switches();
// Immutable per-device properties (cached per device).
struct DevProps {
  int sms, smem_optin;
};
cudaError_t dev_props(DevProps *out);
// Opt a kernel in to `bytes` of dynamic shared memory on the CURRENT device
// (per device and thread-safe: cudaFuncSetAttribute applies to one device).
cudaError_t ensure_dyn_smem(const void *func, int bytes);

constexpr int kMaxSeqs = 2048;  // plan arrays live in shared memory
constexpr int kMaxGroup = 16;   // GQA rows per MMA tile
constexpr int kMaxKvHeads = 128; // per rank; sizes the fixed counter region of the workspace
constexpr int kMaxEntries = 16384; // general-map append: per-request prefix table in shared memory

}  // namespace bkv
