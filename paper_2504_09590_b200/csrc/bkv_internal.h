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
};
int prefill_smem_bytes(int head_dim);
bool prefill_uses_tc(int head_dim);   // tcgen05 kernel (wants 1-half TMA boxes)
cudaError_t launch_prefill(const CUtensorMap &tmK, const CUtensorMap &tmV, const PrefillParams &p,
                           int head_dim, int max_q_len, cudaStream_t s);
cudaError_t launch_prefill_tc(const CUtensorMap &tmK, const CUtensorMap &tmV, const PrefillParams &p,
                              int max_q_len, cudaStream_t s);

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

constexpr int kMaxSeqs = 2048;  // plan arrays live in shared memory
constexpr int kMaxGroup = 16;   // GQA rows per MMA tile
constexpr int kMaxKvHeads = 128; // per rank; sizes the fixed counter region of the workspace
constexpr int kMaxEntries = 16384; // general-map append: per-request prefix table in shared memory

}  // namespace bkv
