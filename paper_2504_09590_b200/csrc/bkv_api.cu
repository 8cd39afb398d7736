// bkv_api.cu -- the C ABI of include/bkv.h: argument checks, TMA descriptor
// encoding, workspace layout, launches, host-side layout validator.
#include <cudaTypedefs.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <map>
#include <mutex>
#include <vector>

#include "../../include/bkv.h"
#include "bkv_internal.h"

namespace bkv {

namespace {
std::mutex g_sw_mu;
DevSwitches g_sw;
std::atomic<bool> g_sw_loaded{false};
int env_int(const char *name, int dflt) {
  const char *s = getenv(name);
  return (s && *s) ? atoi(s) : dflt;
}
void load_switches() {
  DevSwitches s;
  s.slots = env_int("BKV_SLOTS", 2);
  s.warps = env_int("BKV_WARPS", 0);
  s.ctas_per_sm = env_int("BKV_CTAS_PER_SM", 1);
  s.units_per_warp = env_int("BKV_UNITS_PER_WARP", 3);
  s.min_split = env_int("BKV_MIN_SPLIT", -1);
  s.small_plan = env_int("BKV_SMALL_PLAN", 1);
  s.streamk = env_int("BKV_STREAMK", 1);
  s.merge_warps = env_int("BKV_MERGE_WARPS", 8);
  s.fused_merge = env_int("BKV_FUSED_MERGE", 0);
  s.kv_combined = env_int("BKV_KV_COMBINED", 1);
  s.mha_cuda_cores = env_int("BKV_MHA_CUDA_CORES", 0);
  s.prefill_mma_sync = env_int("BKV_PREFILL_MMA_SYNC", 0);
  s.prefill_qt = env_int("BKV_PREFILL_QT", 2);
  s.prefill_q_ldg = env_int("BKV_PREFILL_Q_LDG", 0);
  s.prefill_o_stg = env_int("BKV_PREFILL_O_STG", 0);
#if defined(BKV_DEV_TRACE) || defined(BKV_DEV_PROBES)
  s.prefill_probe = env_int("BKV_PREFILL_PROBE", 0);   // work-skipping what-if probes: dev builds only
#else
  s.prefill_probe = 0;
#endif
  s.mixed_overlap = env_int("BKV_MIXED_OVERLAP", 1);
  s.mixed_reserve = env_int("BKV_MIXED_RESERVE", 24);
#ifdef BKV_DEV_TRACE
  s.debug = env_int("BKV_DEBUG", 0);
  s.trace = env_int("BKV_TRACE", 0);
#else
  s.debug = 0;   // work-skipping probes exist only in the dev trace build
  s.trace = 0;
#endif
  s.planned_slots = env_int("BKV_PLANNED_SLOTS", 2);
  s.planned_dynamic_p = env_int("BKV_PLANNED_DYNAMIC_P", 128);
  s.planned_pf = env_int("BKV_PLANNED_PF", 3);
  g_sw = s;
}
}  // namespace

const DevSwitches &dev_switches() {
  if (!g_sw_loaded.load(std::memory_order_acquire)) {
    std::lock_guard<std::mutex> lk(g_sw_mu);
    if (!g_sw_loaded.load(std::memory_order_relaxed)) {
      load_switches();
      g_sw_loaded.store(true, std::memory_order_release);
    }
  }
  return g_sw;
}

cudaError_t dev_props(DevProps *out) {
  static std::mutex mu;
  static std::map<int, DevProps> cache;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(dev);
  if (it == cache.end()) {
    DevProps d;
    if ((e = cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&d.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev)) != cudaSuccess)
      return e;
    it = cache.emplace(dev, d).first;
  }
  *out = it->second;
  return cudaSuccess;
}

cudaError_t ensure_dyn_smem(const void *func, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void *, int>, int> granted;   // (kernel, device) -> bytes
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  int &have = granted[std::make_pair(func, dev)];
  if (bytes <= have) return cudaSuccess;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}

}  // namespace bkv

namespace {

thread_local char g_err[512] = "";

bkv_status fail(bkv_status s, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
bkv_status fail(bkv_status s, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return s;
}

bkv_status cuda_fail(cudaError_t e, const char *what) {
  return fail(BKV_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

bkv_status check_pool(const bkv_kv_pool *pool) {
  if (!pool) return fail(BKV_ERR_INVALID_ARGUMENT, "pool is NULL");
  if (!pool->k || !pool->v) return fail(BKV_ERR_INVALID_ARGUMENT, "pool k/v pointer is NULL");
  if (pool->head_dim != 64 && pool->head_dim != 128)
    return fail(BKV_ERR_UNSUPPORTED, "head_dim %d not in {64, 128}", pool->head_dim);
  if (pool->block_size != 16 && pool->block_size != 32)
    return fail(BKV_ERR_UNSUPPORTED, "block_size %d not in {16, 32}", pool->block_size);
  if (pool->num_blocks <= 0 || pool->num_kv_heads <= 0)
    return fail(BKV_ERR_INVALID_ARGUMENT, "num_blocks/num_kv_heads must be positive");
  if (!aligned16(pool->k) || !aligned16(pool->v))
    return fail(BKV_ERR_INVALID_ARGUMENT, "pool k/v must be 16-byte aligned");
  if (pool->stride_block % 8 || pool->stride_head % 8 || pool->stride_slot % 8 ||
      pool->stride_block <= 0 || pool->stride_head <= 0 || pool->stride_slot < pool->head_dim)
    return fail(BKV_ERR_INVALID_ARGUMENT,
                "pool strides must be positive multiples of 8 elements with stride_slot >= head_dim");
  return BKV_OK;
}

bkv_status check_map(const bkv_block_map *map) {
  if (!map) return fail(BKV_ERR_INVALID_ARGUMENT, "block map is NULL");
  if (map->num_seqs < 0) return fail(BKV_ERR_INVALID_ARGUMENT, "num_seqs < 0");
  if (map->num_seqs > 0 && (!map->block_tables || !map->dirs))
    return fail(BKV_ERR_INVALID_ARGUMENT, "block_tables/dirs is NULL");
  if (map->bt_stride <= 0) return fail(BKV_ERR_INVALID_ARGUMENT, "bt_stride must be positive");
  if (map->dir_row_stride < 0 || map->dir_col_stride < 0)
    return fail(BKV_ERR_INVALID_ARGUMENT, "direction strides must be >= 0");
  if (map->fills) {   // general map
    if (map->num_seqs > 0 && !map->num_entries)
      return fail(BKV_ERR_INVALID_ARGUMENT, "general map: num_entries is NULL");
    if (map->fill_row_stride < 0)
      return fail(BKV_ERR_INVALID_ARGUMENT, "general map: fill_row_stride < 0");
  }
  return BKV_OK;
}

// ----------------------------------------------------------- TMA descriptors
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 5-D view (64 d, slot, d-half, head, block) of one pool tensor.  The d-half
// dimension (stride 128 B) lets ONE box {64, 16, d/64, 1, 1} fetch a whole
// 16-slot x d tile, landing as [half][slot][128 B] with the 128-byte swizzle
// the decode kernel's ldmatrix / LDS reads are conflict-free against.
bkv_status encode_pool_map(CUtensorMap *m, void *base, const bkv_kv_pool *pool, bool one_half = false) {
  auto fn = encode_fn();
  if (!fn) return fail(BKV_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
  const int halves = pool->head_dim / 64;
  cuuint64_t dims[5] = {64, (cuuint64_t)pool->block_size, (cuuint64_t)halves,
                        (cuuint64_t)pool->num_kv_heads, (cuuint64_t)pool->num_blocks};
  cuuint64_t strides[4] = {(cuuint64_t)pool->stride_slot * 2, 128,
                           (cuuint64_t)pool->stride_head * 2, (cuuint64_t)pool->stride_block * 2};
  cuuint32_t box[5] = {64, 16, one_half ? 1u : (cuuint32_t)halves, 1, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, base, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(BKV_ERR_CUDA, "cuTensorMapEncodeTiled failed (CUresult %d)", (int)r);
  return BKV_OK;
}

// 4-D view (64 d, d-half, q head, token) of the query (or output) rows of the
// prefill kernel: one box {64, 1, g, rows/g} is one 64-d half of `rows` rows
// (rows = (token, head of the group) pairs), 128B-swizzled.  The token extent is
// open-ended (the caller passes no row count): the kernel's tiles end at a
// request's last row, so a box never starts past a token the caller owns, reads
// before token 0 zero-fill, and output boxes hold only the request's own rows.
bkv_status encode_rows_map(CUtensorMap *m, const void *q, int head_dim, int num_q_heads, int64_t st_tok,
                           int64_t st_head, int g, int rows) {
  auto fn = encode_fn();
  if (!fn) return fail(BKV_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
  cuuint64_t dims[4] = {64, (cuuint64_t)(head_dim / 64), (cuuint64_t)num_q_heads, (cuuint64_t)1 << 31};
  cuuint64_t strides[3] = {128, (cuuint64_t)st_head * 2, (cuuint64_t)st_tok * 2};
  cuuint32_t box[4] = {64, 1, (cuuint32_t)g, (cuuint32_t)(rows / g)};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(q), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(BKV_ERR_CUDA, "cuTensorMapEncodeTiled (queries) failed (CUresult %d)", (int)r);
  return BKV_OK;
}

// Combined view of K and V (decode): when the pool is contiguous over (block,
// head) and V sits a multiple of 16 bytes away from K, one 5-D box
// {64 d, 16 slots, d/64 halves, 2 (K, V), 1 (block*H + head)} fetches both
// tiles of a chunk -- one TMA instruction per chunk instead of two.
// Returns 0 (not applicable), 1 (K first) or 2 (V first, V below K).
int encode_pool_map_kv(CUtensorMap *m, const bkv_kv_pool *pool) {
  if (bkv::dev_switches().kv_combined == 0) return 0;
  auto fn = encode_fn();
  if (!fn) return 0;
  if (pool->stride_block != (int64_t)pool->num_kv_heads * pool->stride_head) return 0;
  const int64_t diff = static_cast<const char *>(pool->v) - static_cast<const char *>(pool->k);
  const int64_t ad = diff < 0 ? -diff : diff;
  if (ad == 0 || (ad & 15) || ad >= (int64_t(1) << 40)) return 0;
  void *base = diff > 0 ? pool->k : pool->v;
  const int halves = pool->head_dim / 64;
  cuuint64_t dims[5] = {64, (cuuint64_t)pool->block_size, (cuuint64_t)halves, 2,
                        (cuuint64_t)pool->num_blocks * pool->num_kv_heads};
  cuuint64_t strides[4] = {(cuuint64_t)pool->stride_slot * 2, 128, (cuuint64_t)ad,
                           (cuuint64_t)pool->stride_head * 2};
  cuuint32_t box[5] = {64, 16, (cuuint32_t)halves, 2, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, base, dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return 0;
  return diff > 0 ? 1 : 2;
}

// ------------------------------------------------------------ workspace
struct WsLayout {
  size_t sched, counters, mcnt, ml, o, trace, total;
  int trace_cap;
  int units_max;
};

size_t up256(size_t x) { return (x + 255) & ~size_t(255); }

bkv_status ws_layout(int B, int Hq, int H, int D, WsLayout *w, bkv::DecodeLaunch *cfg, int *slots,
                     int *qb) {
  const int g = Hq / H;
  cudaError_t e = bkv::decode_config(D, g, B, cfg, slots, qb);
  if (e != cudaSuccess) return cuda_fail(e, "querying the device");
  const long long units = (long long)bkv::decode_target_units(*cfg) + (long long)B * H;
  if (units > (1ll << 30)) return fail(BKV_ERR_INVALID_ARGUMENT, "problem too large");
  w->units_max = (int)units;
  // Region A: scheduler words (re-armed to 0 by every call: merge kernel or last CTA),
  // the published split plan; fixed size for every geometry.  Region B
  // (partials) is scratch.
  w->sched = 0;
  w->counters = 256;
  w->mcnt = w->counters + up256((size_t)bkv::kMaxSeqs * bkv::kMaxKvHeads * 4);
  w->ml = w->mcnt + up256((size_t)bkv::kMaxSeqs * bkv::kMaxKvHeads * 4);
  w->o = w->ml + up256((size_t)units * g * 2 * 4);
  w->trace = w->o + up256((size_t)units * g * D * 4);
  w->trace_cap = bkv::dev_switches().trace;   // dev only (trace build): per-warp event log after the partials
  w->total = w->trace + up256((size_t)cfg->grid * cfg->warps * w->trace_cap * 16);
  return BKV_OK;
}

}  // namespace

extern "C" {

const char *bkv_status_string(bkv_status s) {
  switch (s) {
    case BKV_OK: return "BKV_OK";
    case BKV_ERR_INVALID_ARGUMENT: return "BKV_ERR_INVALID_ARGUMENT";
    case BKV_ERR_UNSUPPORTED: return "BKV_ERR_UNSUPPORTED";
    case BKV_ERR_WORKSPACE_TOO_SMALL: return "BKV_ERR_WORKSPACE_TOO_SMALL";
    case BKV_ERR_LAYOUT: return "BKV_ERR_LAYOUT";
    case BKV_ERR_CUDA: return "BKV_ERR_CUDA";
  }
  return "BKV_ERR_UNKNOWN";
}

const char *bkv_last_error(void) { return g_err; }

int32_t bkv_version(void) { return 300; }

static bkv_status append_impl(const bkv_kv_pool *pool, const bkv_block_map *map,
                              const int32_t *seq_lens_before, const int32_t *cu_new_tokens,
                              int32_t total_new_tokens, const void *k_new, const void *v_new,
                              int64_t *slot_mapping_out, const int32_t *evict_rows, void *ckpt_k,
                              void *ckpt_v, bkv_stream_t stream) {
  bkv_status s = check_pool(pool);
  if (s) return s;
  if ((s = check_map(map))) return s;
  if (map->num_seqs == 0 || total_new_tokens == 0) return BKV_OK;
  if (total_new_tokens < 0) return fail(BKV_ERR_INVALID_ARGUMENT, "total_new_tokens < 0");
  if (!seq_lens_before || !cu_new_tokens || !k_new || !v_new)
    return fail(BKV_ERR_INVALID_ARGUMENT, "seq_lens_before/cu_new_tokens/k_new/v_new is NULL");
  if (!aligned16(k_new) || !aligned16(v_new))
    return fail(BKV_ERR_INVALID_ARGUMENT, "k_new/v_new must be 16-byte aligned");
  if (pool->stride_slot != pool->head_dim && pool->stride_slot % 8)
    return fail(BKV_ERR_INVALID_ARGUMENT, "stride_slot");
  bkv::AppendParams p;
  p.k = static_cast<uint16_t *>(pool->k);
  p.v = static_cast<uint16_t *>(pool->v);
  p.sb = pool->stride_block;
  p.sh = pool->stride_head;
  p.ss = pool->stride_slot;
  p.H = pool->num_kv_heads;
  p.bs = pool->block_size;
  p.bt = map->block_tables;
  p.bt_stride = map->bt_stride;
  p.dirs = map->dirs;
  p.dir_rs = map->dir_row_stride;
  p.dir_cs = map->dir_col_stride;
  p.before = seq_lens_before;
  p.cu_new = cu_new_tokens;
  p.k_new = static_cast<const uint16_t *>(k_new);
  p.v_new = static_cast<const uint16_t *>(v_new);
  p.slot_mapping = slot_mapping_out;
  p.B = map->num_seqs;
  p.fills = map->fills;
  p.fill_rs = map->fill_row_stride;
  p.nent = map->num_entries;
  p.max_entries = map->bt_stride;
  if (p.fills && map->bt_stride > bkv::kMaxEntries)
    return fail(BKV_ERR_UNSUPPORTED, "general map: bt_stride %d > %d", map->bt_stride, bkv::kMaxEntries);
  p.evict = evict_rows;
  p.ck_k = static_cast<uint16_t *>(ckpt_k);
  p.ck_v = static_cast<uint16_t *>(ckpt_v);
  cudaError_t e = bkv::launch_kv_append(p, pool->head_dim, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "kv_append launch");
  return BKV_OK;
}

bkv_status bkv_kv_append(const bkv_kv_pool *pool, const bkv_block_map *map,
                         const int32_t *seq_lens_before, const int32_t *cu_new_tokens,
                         int32_t total_new_tokens, const void *k_new, const void *v_new,
                         int64_t *slot_mapping_out, bkv_stream_t stream) {
  return append_impl(pool, map, seq_lens_before, cu_new_tokens, total_new_tokens, k_new, v_new,
                     slot_mapping_out, nullptr, nullptr, nullptr, stream);
}

bkv_status bkv_kv_append_checkpoint(const bkv_kv_pool *pool, const bkv_block_map *map,
                                    const int32_t *seq_lens_before, const int32_t *cu_new_tokens,
                                    int32_t total_new_tokens, const void *k_new, const void *v_new,
                                    int64_t *slot_mapping_out, const int32_t *evict_rows,
                                    void *ckpt_k, void *ckpt_v, bkv_stream_t stream) {
  if (total_new_tokens > 0 && map && map->num_seqs > 0) {
    if (!evict_rows || !ckpt_k || !ckpt_v)
      return fail(BKV_ERR_INVALID_ARGUMENT, "evict_rows/ckpt_k/ckpt_v is NULL");
    if (!aligned16(ckpt_k) || !aligned16(ckpt_v))
      return fail(BKV_ERR_INVALID_ARGUMENT, "ckpt_k/ckpt_v must be 16-byte aligned");
  }
  return append_impl(pool, map, seq_lens_before, cu_new_tokens, total_new_tokens, k_new, v_new,
                     slot_mapping_out, evict_rows, ckpt_k, ckpt_v, stream);
}

static bkv_status slot_copy(const bkv_kv_pool *pool, const int64_t *slot_ids, int32_t n, void *kb,
                            void *vb, int restore, bkv_stream_t stream) {
  bkv_status s = check_pool(pool);
  if (s) return s;
  if (n < 0) return fail(BKV_ERR_INVALID_ARGUMENT, "n < 0");
  if (n == 0) return BKV_OK;
  if (!slot_ids || !kb || !vb) return fail(BKV_ERR_INVALID_ARGUMENT, "slot_ids/buffers is NULL");
  if (!aligned16(kb) || !aligned16(vb)) return fail(BKV_ERR_INVALID_ARGUMENT, "buffers must be 16-byte aligned");
  bkv::SlotCopyParams p;
  p.k = static_cast<uint16_t *>(pool->k);
  p.v = static_cast<uint16_t *>(pool->v);
  p.sb = pool->stride_block;
  p.sh = pool->stride_head;
  p.ss = pool->stride_slot;
  p.H = pool->num_kv_heads;
  p.bs = pool->block_size;
  p.slots = slot_ids;
  p.n = n;
  p.buf_k = static_cast<uint16_t *>(kb);
  p.buf_v = static_cast<uint16_t *>(vb);
  p.restore = restore;
  cudaError_t e = bkv::launch_slot_copy(p, pool->head_dim, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, restore ? "kv_restore launch" : "kv_checkpoint launch");
  return BKV_OK;
}

bkv_status bkv_kv_checkpoint(const bkv_kv_pool *pool, const int64_t *slot_ids, int32_t n, void *k_out,
                             void *v_out, bkv_stream_t stream) {
  return slot_copy(pool, slot_ids, n, k_out, v_out, 0, stream);
}

bkv_status bkv_kv_restore(const bkv_kv_pool *pool, const int64_t *slot_ids, int32_t n, const void *k_in,
                          const void *v_in, bkv_stream_t stream) {
  return slot_copy(pool, slot_ids, n, const_cast<void *>(k_in), const_cast<void *>(v_in), 1, stream);
}

size_t bkv_decode_workspace_size(int32_t num_seqs, int32_t num_q_heads, int32_t num_kv_heads,
                                 int32_t head_dim) {
  if (head_dim != 64 && head_dim != 128) {
    fail(BKV_ERR_UNSUPPORTED, "BKV_ERR_UNSUPPORTED: head_dim %d not in {64, 128}", head_dim);
    return 0;
  }
  if (num_seqs < 0 || num_kv_heads <= 0 || num_q_heads <= 0 || num_q_heads % num_kv_heads) {
    fail(BKV_ERR_INVALID_ARGUMENT,
         "BKV_ERR_INVALID_ARGUMENT: num_q_heads %d must be a positive multiple of num_kv_heads %d",
         num_q_heads, num_kv_heads);
    return 0;
  }
  WsLayout w;
  bkv::DecodeLaunch cfg;
  int slots, qb;
  if (ws_layout(num_seqs, num_q_heads, num_kv_heads, head_dim, &w, &cfg, &slots, &qb)) return 0;
  return w.total;
}

bkv_status bkv_paged_decode_attention(const bkv_kv_pool *pool, const bkv_block_map *map,
                                      const int32_t *seq_lens, int32_t max_seq_len,
                                      const void *q, int64_t q_stride_seq, int64_t q_stride_head,
                                      int32_t num_q_heads, float softmax_scale, void *out,
                                      int64_t o_stride_seq, int64_t o_stride_head, void *workspace,
                                      size_t workspace_bytes, bkv_stream_t stream) {
  return bkv_paged_decode_attention_ex(pool, map, seq_lens, max_seq_len, q, q_stride_seq,
                                       q_stride_head, num_q_heads, softmax_scale, out, o_stride_seq,
                                       o_stride_head, workspace, workspace_bytes, 0u, stream);
}

// Shared by bkv_paged_decode_attention_ex (k_new == v_new == NULL) and
// bkv_decode_step (the fused append of each request's token L-1).
static bkv_status decode_impl(const bkv_kv_pool *pool, const bkv_block_map *map,
                              const int32_t *seq_lens, int32_t max_seq_len, const void *k_new,
                              const void *v_new, const void *q, int64_t q_stride_seq,
                              int64_t q_stride_head, int32_t num_q_heads, float softmax_scale,
                              void *out, int64_t o_stride_seq, int64_t o_stride_head,
                              void *workspace, size_t workspace_bytes, uint32_t flags,
                              bkv_stream_t stream, void *const *peer_outs = nullptr,
                              int32_t n_peers = 0, bool after_own_prefill = false) {
  if (flags & ~(BKV_FLAG_PDL | BKV_FLAG_PEER_MULTICAST))
    return fail(BKV_ERR_INVALID_ARGUMENT, "unknown flags 0x%x", flags);
  if ((flags & BKV_FLAG_PEER_MULTICAST) && n_peers != 1)
    return fail(BKV_ERR_INVALID_ARGUMENT, "BKV_FLAG_PEER_MULTICAST needs exactly one peer output (the multicast address)");
  bkv_status s = check_pool(pool);
  if (s) return s;
  if ((s = check_map(map))) return s;
  const int B = map->num_seqs, H = pool->num_kv_heads, D = pool->head_dim;
  if (B == 0) return BKV_OK;
  if (B > bkv::kMaxSeqs) return fail(BKV_ERR_UNSUPPORTED, "num_seqs %d > %d", B, bkv::kMaxSeqs);
  if (H > bkv::kMaxKvHeads)
    return fail(BKV_ERR_UNSUPPORTED, "num_kv_heads %d > %d", H, bkv::kMaxKvHeads);
  if (!seq_lens || !q || !out || !workspace)
    return fail(BKV_ERR_INVALID_ARGUMENT, "seq_lens/q/out/workspace is NULL");
  if (num_q_heads <= 0 || num_q_heads % H)
    return fail(BKV_ERR_INVALID_ARGUMENT, "num_q_heads %d is not a multiple of num_kv_heads %d",
                num_q_heads, H);
  const int g = num_q_heads / H;
  if (g > bkv::kMaxGroup) return fail(BKV_ERR_UNSUPPORTED, "group %d > %d", g, bkv::kMaxGroup);
  if (max_seq_len < 0 || (int64_t)max_seq_len > (int64_t)map->bt_stride * pool->block_size)
    return fail(BKV_ERR_INVALID_ARGUMENT, "max_seq_len %d exceeds bt_stride*block_size", max_seq_len);
  if (!aligned16(q) || !aligned16(out) || q_stride_seq % 8 || q_stride_head % 8 ||
      o_stride_seq % 8 || o_stride_head % 8)
    return fail(BKV_ERR_INVALID_ARGUMENT, "q/out must be 16-byte aligned with strides multiple of 8");
  if (!(softmax_scale == softmax_scale) || isinf(softmax_scale))
    return fail(BKV_ERR_INVALID_ARGUMENT, "softmax_scale must be finite");
  if ((reinterpret_cast<uintptr_t>(workspace) & 255u) != 0)
    return fail(BKV_ERR_INVALID_ARGUMENT, "workspace must be 256-byte aligned");
  WsLayout w;
  bkv::DecodeLaunch cfg;
  int slots, qb;
  if ((s = ws_layout(B, num_q_heads, H, D, &w, &cfg, &slots, &qb))) return s;
  if (workspace_bytes < w.total)
    return fail(BKV_ERR_WORKSPACE_TOO_SMALL, "workspace %zu < required %zu bytes", workspace_bytes,
                w.total);
  CUtensorMap tmK, tmV;
  if ((s = encode_pool_map(&tmK, pool->k, pool))) return s;
  if ((s = encode_pool_map(&tmV, pool->v, pool))) return s;
  CUtensorMap tmKV;
  const int kv_mode = encode_pool_map_kv(&tmKV, pool);
  if (kv_mode) tmK = tmKV;   // the kernel then issues one box per chunk from tmK
  uint8_t *ws = static_cast<uint8_t *>(workspace);
  bkv::DecodeParams p;
  p.bt = map->block_tables;
  p.bt_stride = map->bt_stride;
  p.dirs = map->dirs;
  p.dir_rs = map->dir_row_stride;
  p.dir_cs = map->dir_col_stride;
  p.seq_lens = seq_lens;
  p.fills = map->fills;
  p.fill_rs = map->fill_row_stride;
  p.nent = map->num_entries;
  p.B = B;
  p.H = H;
  p.bs = pool->block_size;
  p.g = g;
  p.q = static_cast<const uint16_t *>(q);
  p.q_ss = q_stride_seq;
  p.q_sh = q_stride_head;
  p.out = static_cast<uint16_t *>(out);
  p.o_ss = o_stride_seq;
  p.o_sh = o_stride_head;
  p.scale_log2 = softmax_scale * 1.4426950408889634f;
  p.sched = reinterpret_cast<int *>(ws + w.sched);
  p.plan_out = reinterpret_cast<int *>(ws + w.counters);
  p.merge_cnt = reinterpret_cast<int *>(ws + w.mcnt);
  p.part_ml = reinterpret_cast<float *>(ws + w.ml);
  p.part_o = reinterpret_cast<float *>(ws + w.o);
  p.target_units = bkv::decode_target_units(cfg);
  p.min_split = bkv::decode_min_split(g);
  const bkv::DevSwitches &sw = bkv::dev_switches();
  p.small_plan = sw.small_plan;
  p.streamk = sw.streamk;   // 0 off, 1 auto, 2 always (dev)
  p.units_max = w.units_max;
  p.slots = slots;
  p.q_bytes = qb;
  p.total_warps = cfg.grid * cfg.warps;
  p.pdl = (flags & BKV_FLAG_PDL) ? 1 : 0;
  // mixed dispatch: the preceding kernel is our own prefill kernel, which
  // writes only the prefill rows of `out` and was itself launched in stream
  // order -- the decode part may run alongside its tail (no grid wait)
  p.pdl_nowait = (p.pdl && after_own_prefill && sw.mixed_overlap != 0) ? 1 : 0;   // dev: 0 = keep the grid wait
  p.k_new = static_cast<const uint16_t *>(k_new);
  p.v_new = static_cast<const uint16_t *>(v_new);
  p.k_pool = static_cast<uint16_t *>(pool->k);
  p.v_pool = static_cast<uint16_t *>(pool->v);
  p.pool_sb = pool->stride_block;
  p.pool_sh = pool->stride_head;
  p.pool_ss = pool->stride_slot;
  if (n_peers < 0 || n_peers > bkv::kMaxPeers)
    return fail(BKV_ERR_UNSUPPORTED, "n_peers %d outside [0, %d]", n_peers, bkv::kMaxPeers);
  p.n_peers = n_peers;
  p.peer_mc = (flags & BKV_FLAG_PEER_MULTICAST) ? 1 : 0;
  // split merge: separate stream-ordered merge_kernel by default; in-kernel last-arriver merge
  // (opt-in, BKV_FUSED_MERGE=1: measured slower -- the last-arriving warp merges all g rows
  // of a GQA group serially at the tail, e.g. Llama-70B TP1 115 -> 149 us per layer)
  p.fused_merge = (n_peers == 0 && sw.fused_merge) ? 1 : 0;
  if (p.fused_merge) p.streamk = 0;   // the in-kernel merge knows only the split plan
  for (int k = 0; k < bkv::kMaxPeers; ++k) {
    p.peer_out[k] = k < n_peers ? static_cast<uint16_t *>(peer_outs[k]) : nullptr;
    if (k < n_peers && (!peer_outs[k] || !aligned16(peer_outs[k])))
      return fail(BKV_ERR_INVALID_ARGUMENT, "peer output %d is NULL or not 16-byte aligned", k);
  }
  p.kv_mode = kv_mode;
  p.debug_flags = sw.debug;
  p.trace_cap = w.trace_cap;
  p.trace = w.trace_cap ? reinterpret_cast<unsigned long long *>(ws + w.trace) : nullptr;
  cudaError_t e = bkv::launch_decode(tmK, tmV, p, D, cfg, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "decode attention launch");
  return BKV_OK;
}

bkv_status bkv_paged_decode_attention_ex(const bkv_kv_pool *pool, const bkv_block_map *map,
                                         const int32_t *seq_lens, int32_t max_seq_len,
                                         const void *q, int64_t q_stride_seq, int64_t q_stride_head,
                                         int32_t num_q_heads, float softmax_scale, void *out,
                                         int64_t o_stride_seq, int64_t o_stride_head,
                                         void *workspace, size_t workspace_bytes, uint32_t flags,
                                         bkv_stream_t stream) {
  return decode_impl(pool, map, seq_lens, max_seq_len, nullptr, nullptr, q, q_stride_seq,
                     q_stride_head, num_q_heads, softmax_scale, out, o_stride_seq, o_stride_head,
                     workspace, workspace_bytes, flags, stream);
}

bkv_status bkv_decode_step(const bkv_kv_pool *pool, const bkv_block_map *map,
                           const int32_t *seq_lens, int32_t max_seq_len, const void *k_new,
                           const void *v_new, const void *q, int64_t q_stride_seq,
                           int64_t q_stride_head, int32_t num_q_heads, float softmax_scale,
                           void *out, int64_t o_stride_seq, int64_t o_stride_head,
                           void *workspace, size_t workspace_bytes, uint32_t flags,
                           bkv_stream_t stream) {
  if (map && map->num_seqs > 0) {
    if (!k_new || !v_new) return fail(BKV_ERR_INVALID_ARGUMENT, "k_new/v_new is NULL");
    if (!aligned16(k_new) || !aligned16(v_new))
      return fail(BKV_ERR_INVALID_ARGUMENT, "k_new/v_new must be 16-byte aligned");
  }
  return decode_impl(pool, map, seq_lens, max_seq_len, k_new, v_new, q, q_stride_seq,
                     q_stride_head, num_q_heads, softmax_scale, out, o_stride_seq, o_stride_head,
                     workspace, workspace_bytes, flags, stream);
}

bkv_status bkv_decode_multi_out(const bkv_kv_pool *pool, const bkv_block_map *map,
                                const int32_t *seq_lens, int32_t max_seq_len, const void *k_new,
                                const void *v_new, const void *q, int64_t q_stride_seq,
                                int64_t q_stride_head, int32_t num_q_heads, float softmax_scale,
                                void *out, void *const *peer_outs, int32_t n_peers,
                                int64_t o_stride_seq, int64_t o_stride_head, void *workspace,
                                size_t workspace_bytes, uint32_t flags, bkv_stream_t stream) {
  if ((k_new == nullptr) != (v_new == nullptr))
    return fail(BKV_ERR_INVALID_ARGUMENT, "k_new and v_new must both be set or both be NULL");
  if (k_new && (!aligned16(k_new) || !aligned16(v_new)))
    return fail(BKV_ERR_INVALID_ARGUMENT, "k_new/v_new must be 16-byte aligned");
  if (n_peers > 0 && !peer_outs) return fail(BKV_ERR_INVALID_ARGUMENT, "peer_outs is NULL");
  if (n_peers < 0 || n_peers > bkv::kMaxPeers)
    return fail(BKV_ERR_UNSUPPORTED, "n_peers %d outside [0, %d]", n_peers, bkv::kMaxPeers);
  return decode_impl(pool, map, seq_lens, max_seq_len, k_new, v_new, q, q_stride_seq,
                     q_stride_head, num_q_heads, softmax_scale, out, o_stride_seq, o_stride_head,
                     workspace, workspace_bytes, flags, stream, peer_outs, n_peers);
}

bkv_status bkv_peer_barrier(uint32_t *const *pads, int32_t n, int32_t rank, uint32_t *counter,
                            uint32_t *err, uint64_t timeout_ns, bkv_stream_t stream) {
  if (n < 1 || n > bkv::kMaxPeers) return fail(BKV_ERR_UNSUPPORTED, "n %d outside [1, 8]", n);
  if (rank < 0 || rank >= n) return fail(BKV_ERR_INVALID_ARGUMENT, "rank %d outside [0, %d)", rank, n);
  if (!pads || !counter || !err) return fail(BKV_ERR_INVALID_ARGUMENT, "pads/counter/err is NULL");
  bkv::PeerBarrierParams p;
  for (int k = 0; k < bkv::kMaxPeers; ++k) {
    p.pads[k] = k < n ? pads[k] : nullptr;
    if (k < n && !pads[k]) return fail(BKV_ERR_INVALID_ARGUMENT, "pad %d is NULL", k);
  }
  p.n = n;
  p.rank = rank;
  p.counter = counter;
  p.err = err;
  p.timeout_ns = timeout_ns;
  cudaError_t e = bkv::launch_peer_barrier(p, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "peer barrier launch");
  return BKV_OK;
}

bkv_status bkv_validate_layout_host(const int32_t *block_tables, int32_t bt_stride,
                                    const uint8_t *dirs, int32_t dir_row_stride,
                                    int32_t dir_col_stride, int32_t num_seqs,
                                    const int32_t *seq_lens, int32_t num_blocks,
                                    int32_t block_size, int32_t require_nonempty,
                                    int64_t info[5]) {
  if (!info) return fail(BKV_ERR_INVALID_ARGUMENT, "info is NULL");
  for (int i = 0; i < 5; ++i) info[i] = 0;
  if (num_seqs < 0 || block_size <= 0 || num_blocks < 0 || bt_stride <= 0)
    return fail(BKV_ERR_INVALID_ARGUMENT, "bad sizes");
  if (num_seqs > 0 && (!block_tables || !dirs || !seq_lens))
    return fail(BKV_ERR_INVALID_ARGUMENT, "NULL input");
  auto entry = [&](int r, int e) { return block_tables[(int64_t)r * bt_stride + e]; };
  auto dir = [&](int r, int e) {
    return dirs[(int64_t)r * dir_row_stride + (int64_t)e * dir_col_stride];
  };
  // I4: ranges
  for (int r = 0; r < num_seqs; ++r) {
    const int64_t L = seq_lens[r];
    if (L < 0 || L > (int64_t)bt_stride * block_size || (require_nonempty && L == 0)) {
      info[0] = 1; info[1] = r; info[2] = -1; info[3] = L;
      return fail(BKV_ERR_LAYOUT, "I4: seq_len %lld of request %d out of range", (long long)L, r);
    }
    const int nb = (int)((L + block_size - 1) / block_size);
    for (int e = 0; e < nb; ++e) {
      if (entry(r, e) < 0 || entry(r, e) >= num_blocks || dir(r, e) > 1) {
        info[0] = 1; info[1] = r; info[2] = e; info[3] = entry(r, e);
        return fail(BKV_ERR_LAYOUT, "I4: entry %d of request %d invalid", e, r);
      }
    }
  }
  // I2: at most one forward and one reversed entry per physical block
  std::vector<int32_t> fwd(num_blocks, -1), rev(num_blocks, -1);
  for (int r = 0; r < num_seqs; ++r) {
    const int nb = (int)((seq_lens[r] + block_size - 1) / block_size);
    for (int e = 0; e < nb; ++e) {
      std::vector<int32_t> &own = dir(r, e) ? rev : fwd;
      const int32_t b = entry(r, e);
      if (own[b] >= 0) {
        info[0] = 3; info[1] = b; info[2] = dir(r, e); info[3] = own[b]; info[4] = r;
        return fail(BKV_ERR_LAYOUT, "I2: block %d has two %s entries", b, dir(r, e) ? "reversed" : "forward");
      }
      own[b] = r;
    }
  }
  // I1: live slots disjoint.  A forward entry with n live tokens covers slots
  // [0, n), a reversed one [bs-n, bs); check occupancy per slot.
  std::vector<int32_t> occ_r((size_t)num_blocks * block_size, -1);
  std::vector<int64_t> occ_t((size_t)num_blocks * block_size, 0);
  for (int r = 0; r < num_seqs; ++r) {
    const int64_t L = seq_lens[r];
    for (int64_t t = 0; t < L; ++t) {
      const int e = (int)(t / block_size), j = (int)(t % block_size);
      const int slot = dir(r, e) ? block_size - 1 - j : j;
      const size_t k = (size_t)entry(r, e) * block_size + slot;
      if (occ_r[k] >= 0) {
        info[0] = 2; info[1] = occ_r[k]; info[2] = occ_t[k]; info[3] = r; info[4] = t;
        return fail(BKV_ERR_LAYOUT, "I1: token %lld of request %d and token %lld of request %d share a slot",
                    (long long)occ_t[k], occ_r[k], (long long)t, r);
      }
      occ_r[k] = r;
      occ_t[k] = t;
    }
  }
  return BKV_OK;
}

namespace {
// sm_reserve: SMs the persistent tcgen05 prefill grid leaves free (the mixed dispatch's
// decode part, PDL-launched right behind it, starts on them at once)
bkv_status prefill_call(const bkv_kv_pool *pool, const bkv_block_map *map, const int32_t *seq_lens,
                        const int32_t *cu_q, int32_t max_q_len, const void *q, int64_t q_stride_tok,
                        int64_t q_stride_head, int32_t num_q_heads, float softmax_scale, void *out,
                        int64_t o_stride_tok, int64_t o_stride_head, bkv_stream_t stream, int sm_reserve) {
  bkv_status s = check_pool(pool);
  if (s) return s;
  if ((s = check_map(map))) return s;
  const int B = map->num_seqs, H = pool->num_kv_heads;
  if (B == 0 || max_q_len == 0) return BKV_OK;
  if (max_q_len < 0) return fail(BKV_ERR_INVALID_ARGUMENT, "max_q_len < 0");
  if (B > 65535 || H > 65535) return fail(BKV_ERR_UNSUPPORTED, "num_seqs/num_kv_heads > 65535");
  if (!seq_lens || !cu_q || !q || !out)
    return fail(BKV_ERR_INVALID_ARGUMENT, "seq_lens/cu_q/q/out is NULL");
  if (num_q_heads <= 0 || num_q_heads % H)
    return fail(BKV_ERR_INVALID_ARGUMENT, "num_q_heads %d is not a multiple of num_kv_heads %d",
                num_q_heads, H);
  if (!aligned16(q) || !aligned16(out) || q_stride_tok % 8 || q_stride_head % 8 ||
      o_stride_tok % 8 || o_stride_head % 8)
    return fail(BKV_ERR_INVALID_ARGUMENT, "q/out must be 16-byte aligned with strides multiple of 8");
  if (!(softmax_scale == softmax_scale) || isinf(softmax_scale))
    return fail(BKV_ERR_INVALID_ARGUMENT, "softmax_scale must be finite");
  CUtensorMap tmK, tmV;
  const bool tc = bkv::prefill_uses_tc(pool->head_dim);   // tcgen05 kernel: one 64-d half per box
  if ((s = encode_pool_map(&tmK, pool->k, pool, tc))) return s;
  if ((s = encode_pool_map(&tmV, pool->v, pool, tc))) return s;
  bkv::PrefillParams p;
  p.bt = map->block_tables;
  p.bt_stride = map->bt_stride;
  p.dirs = map->dirs;
  p.dir_rs = map->dir_row_stride;
  p.dir_cs = map->dir_col_stride;
  p.fills = map->fills;
  p.fill_rs = map->fill_row_stride;
  p.nent = map->num_entries;
  p.seq_lens = seq_lens;
  p.cu_q = cu_q;
  p.B = B;
  p.H = H;
  p.bs = pool->block_size;
  p.g = num_q_heads / H;
  p.q = static_cast<const uint16_t *>(q);
  p.q_st = q_stride_tok;
  p.q_sh = q_stride_head;
  p.out = static_cast<uint16_t *>(out);
  p.o_st = o_stride_tok;
  p.o_sh = o_stride_head;
  p.scale_log2 = softmax_scale * 1.4426950408889634f;
  p.tiles_max = 0;
  p.q_tma = 0;
  p.sm_reserve = sm_reserve;
  p.probe = bkv::dev_switches().prefill_probe;
  // tcgen05 kernel: Q tiles by TMA when a 128-row tile is whole tokens (g | 128)
  // and output rows by TMA store when a warp's 32 rows are whole tokens (g | 32)
  CUtensorMap tmQ, tmO;
  const bool q_tma = tc && 128 % p.g == 0 && bkv::dev_switches().prefill_q_ldg == 0;
  const bool o_tma = tc && 32 % p.g == 0 && bkv::dev_switches().prefill_o_stg == 0;
  if (q_tma && (s = encode_rows_map(&tmQ, q, pool->head_dim, num_q_heads, q_stride_tok, q_stride_head, p.g, 128)))
    return s;
  if (o_tma && (s = encode_rows_map(&tmO, out, pool->head_dim, num_q_heads, o_stride_tok, o_stride_head, p.g, 32)))
    return s;
  cudaError_t e = bkv::launch_prefill(tmK, tmV, q_tma ? &tmQ : nullptr, o_tma ? &tmO : nullptr, p, pool->head_dim,
                                      max_q_len,
                                      reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "prefill attention launch");
  return BKV_OK;
}

}  // namespace

bkv_status bkv_paged_prefill_attention(const bkv_kv_pool *pool, const bkv_block_map *map,
                                       const int32_t *seq_lens, const int32_t *cu_q,
                                       int32_t max_q_len, const void *q, int64_t q_stride_tok,
                                       int64_t q_stride_head, int32_t num_q_heads,
                                       float softmax_scale, void *out, int64_t o_stride_tok,
                                       int64_t o_stride_head, bkv_stream_t stream) {
  return prefill_call(pool, map, seq_lens, cu_q, max_q_len, q, q_stride_tok, q_stride_head, num_q_heads,
                      softmax_scale, out, o_stride_tok, o_stride_head, stream, 0);
}

bkv_status bkv_paged_mixed_attention(const bkv_kv_pool *pool, const bkv_block_map *map,
                                     const int32_t *seq_lens, const int32_t *cu_q,
                                     int32_t num_prefill_seqs, int32_t num_prefill_rows,
                                     int32_t max_q_len, int32_t max_seq_len, const void *q,
                                     int64_t q_stride_tok, int64_t q_stride_head,
                                     int32_t num_q_heads, float softmax_scale, void *out,
                                     int64_t o_stride_tok, int64_t o_stride_head, void *workspace,
                                     size_t workspace_bytes, uint32_t flags, bkv_stream_t stream) {
  bkv_status s = check_map(map);
  if (s) return s;
  const int B = map->num_seqs;
  if (num_prefill_seqs < 0 || num_prefill_seqs > B || num_prefill_rows < 0)
    return fail(BKV_ERR_INVALID_ARGUMENT, "num_prefill_seqs %d / num_prefill_rows %d out of range",
                num_prefill_seqs, num_prefill_rows);
  if (!aligned16(q) || !aligned16(out) || q_stride_tok % 8 || o_stride_tok % 8)
    return fail(BKV_ERR_INVALID_ARGUMENT, "q/out must be 16-byte aligned with strides multiple of 8");
  // part 1: prefill requests [0, P) -- the causal kernel
  bkv_block_map mp = *map;
  mp.num_seqs = num_prefill_seqs;
  if (num_prefill_seqs > 0 && max_q_len > 0) {
    // a decode-heavy batch (the usual serving iteration): the persistent prefill grid
    // leaves mixed_reserve SMs (24 by default) to the PDL-launched decode part, which
    // streams HBM on them while the prefill computes (Llama-70B TP1 bench batch, 16
    // prefills + 240 decodes: 505 -> 540 TF/s; the TP8 shard, 8x fewer prefill items,
    // loses 2 %: kept at 0); otherwise the decode waits for SMs
    // (only when the prefill has work items enough to spare the SMs: >= 8 per SM)
    const bool decode_heavy = B - num_prefill_seqs >= 4 * num_prefill_seqs;
    int reserve = 0;
    if ((flags & BKV_FLAG_PDL) && decode_heavy && pool && pool->num_kv_heads > 0) {
      bkv::DevProps dp;
      const int64_t g = num_q_heads / pool->num_kv_heads;
      const int64_t items = ((int64_t)num_prefill_rows * g + 255) / 256 * pool->num_kv_heads;   // 2 x 128 rows
      if (bkv::dev_props(&dp) == cudaSuccess && items >= 8LL * dp.sms) reserve = bkv::dev_switches().mixed_reserve;
    }
    s = prefill_call(pool, &mp, seq_lens, cu_q, max_q_len, q, q_stride_tok, q_stride_head, num_q_heads,
                     softmax_scale, out, o_stride_tok, o_stride_head, stream, reserve);
    if (s) return s;
  }
  // part 2: decode requests [P, B), one query row each at rows num_prefill_rows + (r - P)
  const int nd = B - num_prefill_seqs;
  if (nd == 0) return BKV_OK;
  bkv_block_map md = *map;
  md.num_seqs = nd;
  md.block_tables = map->block_tables + (int64_t)num_prefill_seqs * map->bt_stride;
  md.dirs = map->dirs + (int64_t)num_prefill_seqs * map->dir_row_stride;
  if (map->fills) {
    md.fills = map->fills + (int64_t)num_prefill_seqs * map->fill_row_stride;
    md.num_entries = map->num_entries + num_prefill_seqs;
  }
  const uint16_t *qd = static_cast<const uint16_t *>(q) + (int64_t)num_prefill_rows * q_stride_tok;
  uint16_t *od = static_cast<uint16_t *>(out) + (int64_t)num_prefill_rows * o_stride_tok;
  return decode_impl(pool, &md, seq_lens + num_prefill_seqs, max_seq_len, nullptr, nullptr, qd,
                     q_stride_tok, q_stride_head, num_q_heads, softmax_scale, od, o_stride_tok,
                     o_stride_head, workspace, workspace_bytes, flags, stream, nullptr, 0, num_prefill_seqs > 0 && max_q_len > 0);
}

bkv_status bkv_validate_block_map_host(const bkv_block_map *map, const int32_t *seq_lens,
                                       int32_t num_blocks, int32_t block_size,
                                       int32_t require_nonempty, int64_t info[5]) {
  if (!map) return fail(BKV_ERR_INVALID_ARGUMENT, "map is NULL");
  if (!map->fills)
    return bkv_validate_layout_host(map->block_tables, map->bt_stride, map->dirs,
                                    map->dir_row_stride, map->dir_col_stride, map->num_seqs,
                                    seq_lens, num_blocks, block_size, require_nonempty, info);
  if (!info) return fail(BKV_ERR_INVALID_ARGUMENT, "info is NULL");
  for (int i = 0; i < 5; ++i) info[i] = 0;
  const int B = map->num_seqs, bt_stride = map->bt_stride;
  if (B < 0 || block_size <= 0 || block_size > 255 || num_blocks < 0 || bt_stride <= 0 ||
      map->fill_row_stride < 0)
    return fail(BKV_ERR_INVALID_ARGUMENT, "bad sizes");
  if (B > 0 && (!map->block_tables || !map->dirs || !map->num_entries || !seq_lens))
    return fail(BKV_ERR_INVALID_ARGUMENT, "NULL input");
  auto entry = [&](int r, int e) { return map->block_tables[(int64_t)r * bt_stride + e]; };
  auto dir = [&](int r, int e) {
    return map->dirs[(int64_t)r * map->dir_row_stride + (int64_t)e * map->dir_col_stride];
  };
  auto fill = [&](int r, int e) { return (int)map->fills[(int64_t)r * map->fill_row_stride + e]; };
  // I4: ranges, fills, lengths = sum of fills
  for (int r = 0; r < B; ++r) {
    const int E = map->num_entries[r];
    if (E < 0 || E > bt_stride) {
      info[0] = 1; info[1] = r; info[2] = -1; info[3] = E;
      return fail(BKV_ERR_LAYOUT, "I4: num_entries %d of request %d out of range", E, r);
    }
    int64_t sum = 0;
    for (int e = 0; e < E; ++e) {
      if (fill(r, e) < 1 || fill(r, e) > block_size) {
        info[0] = 1; info[1] = r; info[2] = e; info[3] = fill(r, e);
        return fail(BKV_ERR_LAYOUT, "I4: fill %d of entry %d of request %d outside [1, %d]",
                    fill(r, e), e, r, block_size);
      }
      if (entry(r, e) < 0 || entry(r, e) >= num_blocks || dir(r, e) > 1) {
        info[0] = 1; info[1] = r; info[2] = e; info[3] = entry(r, e);
        return fail(BKV_ERR_LAYOUT, "I4: entry %d of request %d invalid", e, r);
      }
      sum += fill(r, e);
    }
    if (sum != seq_lens[r] || (require_nonempty && seq_lens[r] == 0)) {
      info[0] = 1; info[1] = r; info[2] = -2; info[3] = seq_lens[r];
      return fail(BKV_ERR_LAYOUT, "I4: seq_len %d of request %d != sum of its fills %lld (or empty)",
                  seq_lens[r], r, (long long)sum);
    }
  }
  // I2: at most one forward and one reversed entry per physical block
  std::vector<int32_t> fwd(num_blocks, -1), rev(num_blocks, -1);
  for (int r = 0; r < B; ++r) {
    for (int e = 0; e < map->num_entries[r]; ++e) {
      std::vector<int32_t> &own = dir(r, e) ? rev : fwd;
      const int32_t b = entry(r, e);
      if (own[b] >= 0) {
        info[0] = 3; info[1] = b; info[2] = dir(r, e); info[3] = own[b]; info[4] = r;
        return fail(BKV_ERR_LAYOUT, "I2: block %d has two %s entries", b, dir(r, e) ? "reversed" : "forward");
      }
      own[b] = r;
    }
  }
  // I1: entry e covers slots [0, n_e) forward or [bs-n_e, bs) reversed
  std::vector<int32_t> occ_r((size_t)num_blocks * block_size, -1);
  std::vector<int64_t> occ_t((size_t)num_blocks * block_size, 0);
  for (int r = 0; r < B; ++r) {
    int64_t t = 0;
    for (int e = 0; e < map->num_entries[r]; ++e) {
      for (int j = 0; j < fill(r, e); ++j, ++t) {
        const int slot = dir(r, e) ? block_size - 1 - j : j;
        const size_t k = (size_t)entry(r, e) * block_size + slot;
        if (occ_r[k] >= 0) {
          info[0] = 2; info[1] = occ_r[k]; info[2] = occ_t[k]; info[3] = r; info[4] = t;
          return fail(BKV_ERR_LAYOUT, "I1: token %lld of request %d and token %lld of request %d share a slot",
                      (long long)occ_t[k], occ_r[k], (long long)t, r);
        }
        occ_r[k] = r;
        occ_t[k] = t;
      }
    }
  }
  return BKV_OK;
}

// ------------------------------------------------------------ planned decode
void bkv_reload_dev_switches(void) {
  std::lock_guard<std::mutex> lk(bkv::g_sw_mu);
  bkv::load_switches();
  bkv::g_sw_loaded.store(true, std::memory_order_release);
}

// SM count a plan is made for: the caller's, or the current device's (0)
static bkv_status plan_sms(int32_t num_sms, int *sms) {
  if (num_sms < 0 || num_sms > 4096) return fail(BKV_ERR_INVALID_ARGUMENT, "num_sms %d outside [0, 4096]", num_sms);
  if (num_sms > 0) {
    *sms = num_sms;
    return BKV_OK;
  }
  bkv::DevProps dp;
  cudaError_t e = bkv::dev_props(&dp);
  if (e != cudaSuccess) return cuda_fail(e, "querying the device (pass num_sms to plan without one)");
  *sms = dp.sms;
  return BKV_OK;
}

size_t bkv_decode_plan_bytes(int32_t num_seqs, int32_t num_kv_heads, int32_t bt_stride, int32_t num_sms) {
  if (num_seqs < 0 || num_kv_heads <= 0 || bt_stride <= 0) {
    fail(BKV_ERR_INVALID_ARGUMENT, "num_seqs < 0, num_kv_heads <= 0 or bt_stride <= 0");
    return 0;
  }
  int sms = 0;
  if (plan_sms(num_sms, &sms)) return 0;
  return 4 * bkv::plan_words_bound(num_seqs, num_kv_heads, bt_stride, sms, bkv::kPlannedWarps);
}

bkv_status bkv_decode_plan(const int32_t *seq_lens, const bkv_block_map *map, int32_t num_kv_heads,
                           int32_t num_q_heads, int32_t head_dim, int32_t block_size, int32_t num_sms, void *plan,
                           size_t plan_bytes, size_t *plan_bytes_used) {
  bkv_status st = check_map(map);
  if (st) return st;
  const int num_seqs = map->num_seqs, bt_stride = map->bt_stride;
  if ((num_seqs > 0 && !seq_lens) || !plan) return fail(BKV_ERR_INVALID_ARGUMENT, "seq_lens/plan is NULL");
  if (num_seqs > bkv::kMaxSeqs) return fail(BKV_ERR_UNSUPPORTED, "num_seqs %d > %d", num_seqs, bkv::kMaxSeqs);
  if (num_kv_heads <= 0 || num_kv_heads > bkv::kMaxKvHeads)
    return fail(BKV_ERR_UNSUPPORTED, "num_kv_heads %d outside [1, %d]", num_kv_heads, bkv::kMaxKvHeads);
  if (num_q_heads <= 0 || num_q_heads % num_kv_heads)
    return fail(BKV_ERR_INVALID_ARGUMENT, "num_q_heads %d is not a multiple of num_kv_heads %d", num_q_heads,
                num_kv_heads);
  const int g = num_q_heads / num_kv_heads;
  if (g > bkv::kMaxGroup) return fail(BKV_ERR_UNSUPPORTED, "group %d > %d", g, bkv::kMaxGroup);
  if (head_dim != 64 && head_dim != 128) return fail(BKV_ERR_UNSUPPORTED, "head_dim %d not in {64, 128}", head_dim);
  if (block_size != 16 && block_size != 32)
    return fail(BKV_ERR_UNSUPPORTED, "block_size %d not in {16, 32}", block_size);
  if (bt_stride > bkv::kMaxEntries)
    return fail(BKV_ERR_UNSUPPORTED, "bt_stride %d outside [1, %d]", bt_stride, bkv::kMaxEntries);
  if ((reinterpret_cast<uintptr_t>(plan) & 15u) != 0) return fail(BKV_ERR_INVALID_ARGUMENT, "plan must be 16-byte aligned");
  int sms = 0;
  if ((st = plan_sms(num_sms, &sms))) return st;
  bkv::HostMap hm;
  hm.bt = map->block_tables;
  hm.bt_stride = bt_stride;
  hm.dirs = map->dirs;
  hm.dir_rs = map->dir_row_stride;
  hm.dir_cs = map->dir_col_stride;
  hm.fills = map->fills;
  hm.fill_rs = map->fill_row_stride;
  hm.nent = map->num_entries;
  size_t used = 0;
  const char *msg = bkv::build_plan(seq_lens, hm, num_seqs, num_kv_heads, g, head_dim, block_size, sms,
                                    bkv::kPlannedWarps, static_cast<int32_t *>(plan), plan_bytes / 4, &used);
  if (plan_bytes_used) *plan_bytes_used = used * 4;
  if (msg) return fail(strstr(msg, "too small") ? BKV_ERR_WORKSPACE_TOO_SMALL : BKV_ERR_INVALID_ARGUMENT,
                       "bkv_decode_plan: %s", msg);
  return BKV_OK;
}

bkv_status bkv_decode_planned(const bkv_kv_pool *pool, const bkv_block_map *map, const int32_t *seq_lens,
                              const void *plan_host, const void *plan_dev, const void *k_new,
                              const void *v_new, const void *q, int64_t q_stride_seq, int64_t q_stride_head,
                              int32_t num_q_heads, float softmax_scale, void *out, int64_t o_stride_seq,
                              int64_t o_stride_head, void *const *peer_outs, int32_t n_peers,
                              void *workspace, size_t workspace_bytes, uint32_t flags, bkv_stream_t stream) {
  if (flags & ~(BKV_FLAG_PDL | BKV_FLAG_KV_EARLY | BKV_FLAG_PEER_MULTICAST))
    return fail(BKV_ERR_INVALID_ARGUMENT, "unknown flags 0x%x", flags);
  if ((flags & BKV_FLAG_PEER_MULTICAST) && n_peers != 1)
    return fail(BKV_ERR_INVALID_ARGUMENT, "BKV_FLAG_PEER_MULTICAST needs exactly one peer output (the multicast address)");
  if ((flags & BKV_FLAG_KV_EARLY) && !(flags & BKV_FLAG_PDL))
    return fail(BKV_ERR_INVALID_ARGUMENT, "BKV_FLAG_KV_EARLY needs BKV_FLAG_PDL");
  bkv_status s = check_pool(pool);
  if (s) return s;
  if ((s = check_map(map))) return s;
  if (!plan_host || !plan_dev) return fail(BKV_ERR_INVALID_ARGUMENT, "plan_host/plan_dev is NULL");
  if ((reinterpret_cast<uintptr_t>(plan_dev) & 15u) != 0)
    return fail(BKV_ERR_INVALID_ARGUMENT, "plan_dev must be 16-byte aligned");
  const bkv::PlanHeader *hd = static_cast<const bkv::PlanHeader *>(plan_host);
  const int B = map->num_seqs, H = pool->num_kv_heads, D = pool->head_dim;
  if (hd->magic != bkv::kPlanMagic || hd->version != bkv::kPlanVersion)
    return fail(BKV_ERR_INVALID_ARGUMENT, "plan_host is not a bkv_decode_plan buffer of this library version");
  if (B == 0) return BKV_OK;
  if ((k_new == nullptr) != (v_new == nullptr))
    return fail(BKV_ERR_INVALID_ARGUMENT, "k_new and v_new must both be set or both be NULL");
  if (k_new && (!aligned16(k_new) || !aligned16(v_new)))
    return fail(BKV_ERR_INVALID_ARGUMENT, "k_new/v_new must be 16-byte aligned");
  if (!seq_lens || !q || !out || !workspace)
    return fail(BKV_ERR_INVALID_ARGUMENT, "seq_lens/q/out/workspace is NULL");
  if (num_q_heads <= 0 || num_q_heads % H)
    return fail(BKV_ERR_INVALID_ARGUMENT, "num_q_heads %d is not a multiple of num_kv_heads %d", num_q_heads, H);
  const int g = num_q_heads / H;
  bkv::DevProps dp;
  cudaError_t e = bkv::dev_props(&dp);
  if (e != cudaSuccess) return cuda_fail(e, "querying the device");
  if (hd->B != B || hd->H != H || hd->g != g || hd->D != D || hd->bs != pool->block_size ||
      hd->general != (map->fills ? 1 : 0) || hd->max_entries > map->bt_stride)
    return fail(BKV_ERR_INVALID_ARGUMENT,
                "plan built for (B %d, H %d, g %d, d %d, bs %d, general %d, entries %d) does not match the call "
                "(B %d, H %d, g %d, d %d, bs %d, general %d, bt_stride %d)",
                hd->B, hd->H, hd->g, hd->D, hd->bs, hd->general, hd->max_entries, B, H, g, D, pool->block_size,
                map->fills ? 1 : 0, map->bt_stride);
  if ((int64_t)B * num_q_heads > (int64_t)bkv::kMaxSeqs * bkv::kMaxKvHeads)
    return fail(BKV_ERR_UNSUPPORTED, "num_seqs x num_q_heads %lld exceeds the workspace's %d row counters",
                (long long)B * num_q_heads, bkv::kMaxSeqs * bkv::kMaxKvHeads);
  if (hd->grid != dp.sms || hd->warps != bkv::kPlannedWarps)
    return fail(BKV_ERR_INVALID_ARGUMENT, "plan built for %d x %d warps, this device runs %d x %d", hd->grid,
                hd->warps, dp.sms, bkv::kPlannedWarps);
  // Large problems (long warp ranges: e.g. OPT-30B at one GPU, 190 blocks per warp) run the
  // dynamically scheduled kernel instead: over a long kernel, per-SM bandwidth differences
  // outweigh the static plan's fixed-cost savings (measured OPT-30B TP1 313 vs 299 us per
  // layer; Llama-70B TP1, 64 blocks per warp, 106 vs 111 for the static plan).
  const int dyn_p = bkv::dev_switches().planned_dynamic_p;
  if (dyn_p > 0 && hd->P >= dyn_p)
    return decode_impl(pool, map, seq_lens, map->bt_stride * pool->block_size, k_new, v_new, q, q_stride_seq,
                       q_stride_head, num_q_heads, softmax_scale, out, o_stride_seq, o_stride_head, workspace,
                       workspace_bytes, flags & (BKV_FLAG_PDL | BKV_FLAG_PEER_MULTICAST), stream, peer_outs,
                       n_peers);
  if (!aligned16(q) || !aligned16(out) || q_stride_seq % 8 || q_stride_head % 8 || o_stride_seq % 8 ||
      o_stride_head % 8)
    return fail(BKV_ERR_INVALID_ARGUMENT, "q/out must be 16-byte aligned with strides multiple of 8");
  if (!(softmax_scale == softmax_scale) || isinf(softmax_scale))
    return fail(BKV_ERR_INVALID_ARGUMENT, "softmax_scale must be finite");
  if ((reinterpret_cast<uintptr_t>(workspace) & 255u) != 0)
    return fail(BKV_ERR_INVALID_ARGUMENT, "workspace must be 256-byte aligned");
  if (n_peers < 0 || n_peers > bkv::kMaxPeers)
    return fail(BKV_ERR_UNSUPPORTED, "n_peers %d outside [0, %d]", n_peers, bkv::kMaxPeers);
  if (n_peers > 0 && !peer_outs) return fail(BKV_ERR_INVALID_ARGUMENT, "peer_outs is NULL");
  WsLayout w;
  bkv::DecodeLaunch cfg;
  int slots0, qb;
  if ((s = ws_layout(B, num_q_heads, H, D, &w, &cfg, &slots0, &qb))) return s;
  if (workspace_bytes < w.total)
    return fail(BKV_ERR_WORKSPACE_TOO_SMALL, "workspace %zu < required %zu bytes", workspace_bytes, w.total);
  if ((size_t)2 * hd->grid * bkv::planned_piece_floats(g, D) * 4 > w.trace - w.o)
    return fail(BKV_ERR_WORKSPACE_TOO_SMALL, "workspace partial region too small for the plan");
  const int S = std::max(1, std::min(4, bkv::dev_switches().planned_slots));
  const int smem = bkv::planned_smem_bytes(D, g, S, hd->warps);
  if (smem > dp.smem_optin) return fail(BKV_ERR_UNSUPPORTED, "planned kernel needs %d B of shared memory", smem);
  CUtensorMap tmK, tmV;
  if ((s = encode_pool_map(&tmK, pool->k, pool))) return s;
  if ((s = encode_pool_map(&tmV, pool->v, pool))) return s;
  CUtensorMap tmKV;
  const int kv_mode = encode_pool_map_kv(&tmKV, pool);
  if (kv_mode) tmK = tmKV;
  uint8_t *ws = static_cast<uint8_t *>(workspace);
  const int32_t *pw = static_cast<const int32_t *>(plan_dev);
  bkv::PlannedParams p;
  p.bt = map->block_tables;
  p.bt_stride = map->bt_stride;
  p.dirs = map->dirs;
  p.dir_rs = map->dir_row_stride;
  p.dir_cs = map->dir_col_stride;
  p.seq_lens = seq_lens;
  p.fills = map->fills;
  p.fill_rs = map->fill_row_stride;
  p.nent = map->num_entries;
  p.B = B;
  p.H = H;
  p.bs = pool->block_size;
  p.g = g;
  p.q = static_cast<const uint16_t *>(q);
  p.q_ss = q_stride_seq;
  p.q_sh = q_stride_head;
  p.out = static_cast<uint16_t *>(out);
  p.o_ss = o_stride_seq;
  p.o_sh = o_stride_head;
  p.scale_log2 = softmax_scale * 1.4426950408889634f;
  p.wseg = pw + hd->off_wseg;
  p.segs = reinterpret_cast<const int4 *>(pw + hd->off_segs);
  p.ctask = pw + hd->off_ctask;
  p.tasks = reinterpret_cast<const int4 *>(pw + hd->off_tasks);
  p.zero = pw + hd->off_zero;
  p.xrows = reinterpret_cast<const int4 *>(pw + hd->off_xrows);
  p.plan_hdr = pw;
  p.ent = reinterpret_cast<const uint32_t *>(pw + hd->off_ent);
  p.xrows_cap = hd->grid;
  p.gpiece = reinterpret_cast<float *>(ws + w.o);
  p.slots = S;
  p.pdl = (flags & BKV_FLAG_PDL) ? 1 : 0;
  p.kv_early = (flags & BKV_FLAG_KV_EARLY) ? 1 : 0;
  p.pf = std::max(0, std::min(32, bkv::dev_switches().planned_pf));
  p.kv_mode = kv_mode;
  p.k_new = static_cast<const uint16_t *>(k_new);
  p.v_new = static_cast<const uint16_t *>(v_new);
  p.k_pool = static_cast<uint16_t *>(pool->k);
  p.v_pool = static_cast<uint16_t *>(pool->v);
  p.pool_sb = pool->stride_block;
  p.pool_sh = pool->stride_head;
  p.pool_ss = pool->stride_slot;
  p.n_peers = n_peers;
  p.peer_mc = (flags & BKV_FLAG_PEER_MULTICAST) ? 1 : 0;
  for (int k = 0; k < bkv::kMaxPeers; ++k) {
    p.peer_out[k] = k < n_peers ? static_cast<uint16_t *>(peer_outs[k]) : nullptr;
    if (k < n_peers && (!peer_outs[k] || !aligned16(peer_outs[k])))
      return fail(BKV_ERR_INVALID_ARGUMENT, "peer output %d is NULL or not 16-byte aligned", k);
  }
  p.trace = w.trace_cap >= 8 ? reinterpret_cast<unsigned long long *>(ws + w.trace) : nullptr;
  e = bkv::launch_planned(tmK, tmV, p, D, hd->grid, hd->warps, smem, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "planned decode launch");
  return BKV_OK;
}

}  // extern "C"
