/*
 * bkv.h -- C ABI of libbkv: BROS bidirectional paged KV cache, B200 (sm_100a).
 *
 * BROS (arXiv 2504.09590) serves real-time (RT) and best-effort (BE) requests
 * from ONE pool of KV blocks: "Each block can be used for KV cache storage of
 * one RT request and one BE request ... the RT request occupies memory slots
 * from the left to the right in the block while that of the BE request in the
 * opposite direction" (§5.1).  The decode kernel is guided by
 * "a binary direction table, which possesses an identical shape to the block
 * tables" and inverts the slot order "whenever the flag of direction is
 * evaluated to be true".  This library exports the two device calls of
 * that hot path:
 *
 *   bkv_kv_append               -- write this step's new K/V rows into their slots
 *   bkv_paged_decode_attention  -- per-request decode attention over the pool
 *
 * and the SURVEY §8(f) rows built on them:
 *
 *   bkv_kv_append_checkpoint, bkv_kv_checkpoint, bkv_kv_restore   (f1 lazy checkpoint)
 *   bkv_decode_step, bkv_decode_multi_out, bkv_peer_barrier       (f2 fused step / reassembly)
 *   bkv_block_map.fills / num_entries in every call               (f3 general maps)
 *   bkv_paged_prefill_attention, bkv_paged_mixed_attention        (f4 mixed prefill + decode)
 *
 * and the planned decode of the same path (host-built split plan, one launch
 * per layer): bkv_decode_plan, bkv_decode_planned; plus host helpers
 * (workspace sizing, host-side layout validators, status strings).
 *
 * Conventions (all entry points):
 *   - Device pointers are caller-owned (allocated by PyTorch or cudaMalloc);
 *     the library never allocates, frees or synchronises.  Every device call is
 *     asynchronous on `stream` and CUDA-graph capturable.
 *   - Argument errors are detected on the host BEFORE any launch and return a
 *     non-zero bkv_status with no side effect; bkv_last_error() then returns a
 *     thread-local one-line explanation.  Launch failures return BKV_ERR_CUDA.
 *     Device-side faults (e.g. a block id out of range that the caller did not
 *     validate) surface asynchronously, as for any CUDA kernel.
 *   - No global mutable state besides per-device caches of immutable device
 *     properties and of kernel shared-memory opt-ins (mutex-guarded), and the
 *     developer switches read once per process: calls are thread-safe.
 *   - Element type of K, V, Q, out, k_new, v_new is bf16 (IEEE bfloat16 bits);
 *     all strides are in ELEMENTS.  Reading Q1: the paper never states the
 *     precision; this library stores bf16 and accumulates in fp32.
 */
#ifndef BKV_H_
#define BKV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define BKV_API __attribute__((visibility("default")))
#else
#define BKV_API
#endif

/* cudaStream_t without pulling in the CUDA headers (same underlying type). */
typedef struct CUstream_st *bkv_stream_t;

/* Direction flag values of the direction table (reading Q4). */
#define BKV_DIR_FWD 0 /* RT: j-th token of a block at slot j             */
#define BKV_DIR_REV 1 /* BE: j-th token of a block at slot block_size-1-j */

typedef enum {
  BKV_OK = 0,
  BKV_ERR_INVALID_ARGUMENT = 1, /* null pointer, bad size/stride/alignment        */
  BKV_ERR_UNSUPPORTED = 2,      /* head_dim/block_size/group outside the built set */
  BKV_ERR_WORKSPACE_TOO_SMALL = 3,
  BKV_ERR_LAYOUT = 4,           /* host validator found an I1-I4 violation         */
  BKV_ERR_CUDA = 5              /* CUDA runtime / driver error                     */
} bkv_status;

/*
 * One layer of one rank's head shard of the KV block pool.
 * Element (block b, kv head h, slot s, dim i) of K lives at
 *     k[b*stride_block + h*stride_head + s*stride_slot + i]      (same for V).
 * Requirements: k, v 16-byte aligned; stride_* multiples of 8 elements;
 * stride_slot >= head_dim; head_dim in {64, 128}; block_size in {16, 32}.
 * Recommended (what the Python binding allocates): contiguous
 * [num_blocks][num_kv_heads][block_size][head_dim], so one (block, head) tile
 * is block_size*head_dim*2 contiguous bytes (4 KiB at bs16/d128).
 */
typedef struct {
  void *k;
  void *v;
  int32_t num_blocks;
  int32_t num_kv_heads;
  int32_t block_size;
  int32_t head_dim;
  int64_t stride_block;
  int64_t stride_head;
  int64_t stride_slot;
} bkv_kv_pool;

/*
 * Block map of a batch (SURVEY D2 + D3).
 *
 * Dense map (fills == NULL, the vLLM-style table the paper's kernel reads):
 * request r's logical token t lives in physical block
 *     block_tables[r*bt_stride + t/block_size]
 * at slot  t%block_size                  if dir == BKV_DIR_FWD
 *          block_size-1-t%block_size     if dir == BKV_DIR_REV
 * where dir = dirs[r*dir_row_stride + (t/block_size)*dir_col_stride].
 * dir_col_stride = 0 gives one flag per request (reading Q5); a table of the
 * block table's shape uses dir_col_stride = 1, dir_row_stride = bt_stride.
 * Only entries e < ceil(seq_len/block_size) are read.
 *
 * General map (fills != NULL, reading Q6 option B):
 * FindBlock places a BE prefill "according to the maximum number of empty
 * slots" and FindPreemptBlock lets an RT request write a BE block
 * "from the opposite end", so ANY entry may be partly filled.
 * Entry e < num_entries[r] of request r holds
 *     n_e = fills[r*fill_row_stride + e]   (1 <= n_e <= block_size)
 * of the request's tokens: tokens are numbered in entry order (entry e holds
 * tokens [n_0+...+n_{e-1}, n_0+...+n_e)) and the j-th token of an entry sits
 * at slot j (forward) or block_size-1-j (reversed) -- the in-block rule of
 * P:711.  The request's resident length is n_0 + ... + n_{num_entries[r]-1};
 * every call that takes seq_lens requires them to be equal (caller
 * precondition, checked by bkv_validate_block_map_host).  A dense map is the
 * general map with every non-last entry full.
 *
 * All pointers are device pointers (host pointers for the host validator).
 */
typedef struct {
  const int32_t *block_tables;
  int32_t bt_stride;
  const uint8_t *dirs;
  int32_t dir_row_stride;
  int32_t dir_col_stride;
  int32_t num_seqs;
  /* general map only (NULL/0 for a dense map) */
  const uint8_t *fills;        /* [num_seqs][fill_row_stride], entries 1..block_size */
  int32_t fill_row_stride;     /* >= num_entries[r] for every r                      */
  const int32_t *num_entries;  /* [num_seqs], 0..bt_stride; required iff fills       */
} bkv_block_map;

/*
 * kv_append -- SURVEY §8(a) row a2: write the K/V rows of this step's new
 * tokens into the pool, each in its request's direction.  RT and BE
 * requests sharing a block write opposite ends in the same launch.
 *
 *   seq_lens_before [num_seqs]   device int32: resident tokens before the append
 *   cu_new_tokens   [num_seqs+1] device int32: new tokens of request r are rows
 *                                cu_new_tokens[r] .. cu_new_tokens[r+1]-1 of
 *                                k_new/v_new (decode step: cu[r] = r)
 *   total_new_tokens             host int: cu_new_tokens[num_seqs]
 *   k_new, v_new                 device bf16 [total_new][num_kv_heads][head_dim],
 *                                contiguous, 16-byte aligned
 *   slot_mapping_out             optional device int64 [total_new]: receives
 *                                block*block_size + slot of every new token
 * The new token t = seq_lens_before[r] + j must lie inside the block map
 * (dense: t < bt_stride*block_size; general: t < the sum of the request's
 * fills -- the map describes the state AFTER the append) and its slot must not
 * hold a live token of another request (invariant I5; lazy-checkpoint
 * eviction is the caller's job).  General maps: num_entries[r] <= 16384.
 * Bit-exact: each written row is a copy of the input row; no other byte of
 * the pool changes.
 */
BKV_API bkv_status bkv_kv_append(const bkv_kv_pool *pool, const bkv_block_map *map,
                         const int32_t *seq_lens_before, const int32_t *cu_new_tokens,
                         int32_t total_new_tokens, const void *k_new, const void *v_new,
                         int64_t *slot_mapping_out, bkv_stream_t stream);

/*
 * paged_decode_attention -- SURVEY §8(a) rows a3-a5.  For every request r and
 * query head h (kv head h / (num_q_heads/num_kv_heads), reading Q9):
 *     out[r][h] = softmax_t(softmax_scale * q[r][h] . K_r[t]) . V_r[t],  t < seq_lens[r]
 * where K_r/V_r are read through the bidirectional block map.  Split-K across
 * the context with an online-softmax merge; fp32 accumulation; output rounded
 * to bf16 (round-to-nearest-even).  The result is permutation-invariant over
 * a request's tokens, so blocks are consumed in physical slot order and the
 * direction only decides which slots of a partly filled block are live.
 *
 *   seq_lens [num_seqs]  device int32, >= 0, includes the token appended this
 *                        step (reading Q7); 0 yields a zero output row (Q8)
 *   max_seq_len          host upper bound of seq_lens (<= bt_stride*block_size)
 *   q                    device bf16, q[r*q_stride_seq + h*q_stride_head + i]
 *   num_q_heads          multiple of pool->num_kv_heads, group <= 16
 *   softmax_scale        e.g. 1/sqrt(head_dim) (reading Q2)
 *   out                  device bf16, out[r*o_stride_seq + h*o_stride_head + i]
 *                        (head-major [H_q][B][d] is o_stride_head = B*d,
 *                        o_stride_seq = d: what the TP all-gather wants)
 *   workspace            device buffer of >= bkv_decode_workspace_size(...) bytes,
 *                        ZERO-FILLED before its first use.  Its synchronisation
 *                        region (scheduler word + per-(request, kv head) split
 *                        counters, fixed size for every geometry) is restored
 *                        to zero by every call, so one workspace serves calls of
 *                        any geometry in sequence -- but never two concurrent
 *                        calls (one workspace per stream).
 *   Limits: num_seqs <= 2048, num_kv_heads <= 128 per call (BKV_ERR_UNSUPPORTED).
 * Deterministic: split partials are merged in split order.
 */
BKV_API bkv_status bkv_paged_decode_attention(const bkv_kv_pool *pool, const bkv_block_map *map,
                                      const int32_t *seq_lens, int32_t max_seq_len,
                                      const void *q, int64_t q_stride_seq, int64_t q_stride_head,
                                      int32_t num_q_heads, float softmax_scale,
                                      void *out, int64_t o_stride_seq, int64_t o_stride_head,
                                      void *workspace, size_t workspace_bytes,
                                      bkv_stream_t stream);

/*
 * Lazy checkpointing.  "Only the KV tensors of a
 * specific request that are about to be overwritten by its peer need to be
 * checkpointed in CPU memory" and are "swapped back into GPU memory when the
 * request is scheduled"; BROS uses "CUDA kernels to
 * efficiently fetch and store KV caches in non-continuous GPU memory".
 *
 *   bkv_kv_checkpoint  gathers the K and V rows (every kv head of the pool) of
 *                      n physical slots -- slot id = block*block_size + slot,
 *                      the value bkv_kv_append reports in slot_mapping_out --
 *                      into k_out / v_out, bf16 [n][num_kv_heads][head_dim]
 *                      contiguous, 16-byte aligned.  The destination may be
 *                      device memory or the device alias of mapped pinned host
 *                      memory (a direct device-to-host checkpoint).
 *   bkv_kv_restore     scatters such rows back into their slots (swap-in).
 * Both are bit-exact copies and change nothing else.  Issue the checkpoint
 * BEFORE the bkv_kv_append that overwrites those slots, on the same stream
 * (stream order is the synchronisation).  Slot ids must be < num_blocks *
 * block_size; n = 0 is a no-op.
 */
BKV_API bkv_status bkv_kv_checkpoint(const bkv_kv_pool *pool, const int64_t *slot_ids, int32_t n,
                                     void *k_out, void *v_out, bkv_stream_t stream);
BKV_API bkv_status bkv_kv_restore(const bkv_kv_pool *pool, const int64_t *slot_ids, int32_t n,
                                  const void *k_in, const void *v_in, bkv_stream_t stream);

/*
 * bkv_kv_append_checkpoint -- kv_append with the lazy checkpoint fused in
 * ("only the KV tensors of a specific request
 * that are about to be overwritten by its peer need to be checkpointed in CPU
 * memory", the a3/B8 example of P:731).  Identical to bkv_kv_append, except:
 *   evict_rows [total_new]  device int32: -1, or the row of ckpt_k/ckpt_v that
 *                           receives the OLD K and V rows (every kv head) of
 *                           new token i's slot before the new rows replace them
 *   ckpt_k, ckpt_v          bf16 [rows][num_kv_heads][head_dim], contiguous,
 *                           16-byte aligned: device memory or the device alias
 *                           of mapped pinned host memory (a direct D2H
 *                           checkpoint)
 * Equal, bit for bit, to bkv_kv_checkpoint of those slots followed by
 * bkv_kv_append; the old row is read and the new one written by the same
 * thread, so no ordering is needed.  Which slots hold live peer tokens is
 * the host scheduler's knowledge (its preemption table).  Rows of
 * ckpt_* not named by evict_rows are not written.
 */
BKV_API bkv_status bkv_kv_append_checkpoint(const bkv_kv_pool *pool, const bkv_block_map *map,
                                            const int32_t *seq_lens_before,
                                            const int32_t *cu_new_tokens, int32_t total_new_tokens,
                                            const void *k_new, const void *v_new,
                                            int64_t *slot_mapping_out, const int32_t *evict_rows,
                                            void *ckpt_k, void *ckpt_v, bkv_stream_t stream);

/*
 * bkv_paged_decode_attention_ex -- the same call with launch flags.
 *   BKV_FLAG_PDL  launch the attention and merge kernels with programmatic
 *                 dependent launch: the split-plan prologue (which reads only
 *                 seq_lens, and num_entries for a general map) overlaps the
 *                 tail of the preceding kernel on the stream, e.g.
 *                 bkv_kv_append or the previous call's merge; both kernels
 *                 trigger their dependents early, so the next kernel's CTAs
 *                 are scheduled as SMs free up.  Contract: seq_lens (and
 *                 num_entries) must NOT be written by the kernel that
 *                 immediately precedes this call on the stream (host copies
 *                 and earlier kernels are fine); every other input is read
 *                 only after that kernel has completed.
 * Unknown flag bits return BKV_ERR_INVALID_ARGUMENT.
 */
#define BKV_FLAG_PDL 1u
/* bkv_decode_planned only, with BKV_FLAG_PDL: the RESIDENT KV of the pool (every
 * token except the ones this call appends) is not written by the immediately
 * preceding kernel either -- true when that kernel is e.g. the layer's QKV
 * projection or another layer's decode call -- so the first tiles of every
 * warp's ring are requested, and its next few blocks prefetched into L2,
 * before the grid wait; q, k_new, v_new and the workspace are still read
 * after it. */
#define BKV_FLAG_KV_EARLY 2u
/* bkv_decode_multi_out and bkv_decode_planned: peer_outs[0] (n_peers must be 1)
 * is an NVLS MULTICAST address (cuMulticastCreate / torch symmetric memory's
 * multicast_ptr) that maps every rank's global output: each output row slice
 * is stored ONCE with multimem.st and the NVSwitch replicates it to every rank
 * bound to the object (PAPER.md P:759 moves these outputs
 * with NCCL).  Same offsets as the per-peer form; completion still needs
 * bkv_peer_barrier (which orders the multicast alias before its release). */
#define BKV_FLAG_PEER_MULTICAST 4u
BKV_API bkv_status bkv_paged_decode_attention_ex(const bkv_kv_pool *pool, const bkv_block_map *map,
                                                 const int32_t *seq_lens, int32_t max_seq_len,
                                                 const void *q, int64_t q_stride_seq,
                                                 int64_t q_stride_head, int32_t num_q_heads,
                                                 float softmax_scale, void *out, int64_t o_stride_seq,
                                                 int64_t o_stride_head, void *workspace,
                                                 size_t workspace_bytes, uint32_t flags,
                                                 bkv_stream_t stream);

/*
 * bkv_decode_step -- one decode iteration of a layer in ONE launch pair
 * (SURVEY §8(f) f2): append each request's newest token and attend over the
 * context that includes it.
 *
 * Defined as exactly
 *     bkv_kv_append(pool, map, seq_lens_before = seq_lens - 1,
 *                   cu_new_tokens = {0, 1, ..., num_seqs}, k_new, v_new, NULL)
 *     bkv_paged_decode_attention_ex(pool, map, seq_lens, ...)
 * i.e. token t = seq_lens[r] - 1 of request r goes to slot
 * (dir ? bs-1-t%bs : t%bs) of block block_tables[r][t / bs] (§5.1,
 * RT fills a block from the left, BE from the right) and the attention
 * then reads it.  Results (pool bytes and out) are bit-identical to the two
 * separate calls.  The warp that owns the 16-slot chunk holding slot(t)
 * bulk-loads the new K/V rows together with that chunk's tile, patches them
 * into the tile in shared memory and bulk-stores them into the pool: no
 * separate append kernel, no extra pool read, no ordering stall.
 *   k_new, v_new  device bf16 [num_seqs][num_kv_heads][head_dim], contiguous,
 *                 16-byte aligned; read only.
 *   seq_lens      device int32 [num_seqs], lengths AFTER the append (>= 1 for
 *                 a request to receive a token; a request with seq_lens 0 is
 *                 left untouched and its output is 0).
 *   the rest      as bkv_paged_decode_attention_ex (same workspace, flags).
 * The map must be valid for lengths seq_lens (I1-I4): the new slot must be
 * free of other requests' live tokens.
 */
BKV_API bkv_status bkv_decode_step(const bkv_kv_pool *pool, const bkv_block_map *map,
                                   const int32_t *seq_lens, int32_t max_seq_len,
                                   const void *k_new, const void *v_new, const void *q,
                                   int64_t q_stride_seq, int64_t q_stride_head,
                                   int32_t num_q_heads, float softmax_scale, void *out,
                                   int64_t o_stride_seq, int64_t o_stride_head, void *workspace,
                                   size_t workspace_bytes, uint32_t flags, bkv_stream_t stream);

/*
 * bkv_decode_multi_out -- decode attention (k_new = v_new = NULL) or the fused
 * decode step (both set, as bkv_decode_step) whose outputs are ALSO stored
 * into n_peers further buffers: the fused reassembly of SURVEY §8(f) row f2.
 * Under tensor parallelism by kv head (outputs moved with NCCL in the
 * paper) every rank writes its head slice straight into every peer's
 * global output over NVLink instead of a separate all-gather.
 *   out          this rank's output (as bkv_paged_decode_attention)
 *   peer_outs    HOST array of n_peers (0..8) device-accessible pointers (peer
 *                memory mapped by CUDA IPC / symmetric memory, or local
 *                buffers); row (r, h) goes to peer_outs[k] + r*o_stride_seq +
 *                h*o_stride_head exactly as to out (callers bake their head-
 *                slice offset into the pointer), 16-byte aligned
 * The peer copies are written by the stream-ordered merge kernel with 8-byte
 * vector stores (bit-identical to out).  Completion is visible to the peers
 * only after bkv_peer_barrier on every rank.
 */
BKV_API bkv_status bkv_decode_multi_out(const bkv_kv_pool *pool, const bkv_block_map *map,
                                        const int32_t *seq_lens, int32_t max_seq_len,
                                        const void *k_new, const void *v_new, const void *q,
                                        int64_t q_stride_seq, int64_t q_stride_head,
                                        int32_t num_q_heads, float softmax_scale, void *out,
                                        void *const *peer_outs, int32_t n_peers,
                                        int64_t o_stride_seq, int64_t o_stride_head,
                                        void *workspace, size_t workspace_bytes, uint32_t flags,
                                        bkv_stream_t stream);

/*
 * bkv_peer_barrier -- stream-ordered cross-rank completion signal for the
 * fused reassembly: rank `rank` of n stores epoch e (device counter *counter,
 * incremented by this call, so graph replays need no host update) into
 * pads[k][rank] for every k (release, system scope) and waits until
 * pads[rank][k] >= e for every k (acquire).  pads = HOST array of n
 * device-accessible uint32 arrays of n entries (zeroed before first use);
 * every rank must call it the same number of times.  A wait longer than
 * timeout_ns (%globaltimer) stops waiting and sets *err = 1 instead of hanging.
 */
BKV_API bkv_status bkv_peer_barrier(uint32_t *const *pads, int32_t n, int32_t rank,
                                    uint32_t *counter, uint32_t *err, uint64_t timeout_ns,
                                    bkv_stream_t stream);

/*
 * bkv_paged_prefill_attention -- mixed prefill + decode attention over the
 * bidirectional paged cache.  BROS batches "the
 * concatenated prefill requests followed by the decode requests" and
 * dispatches each part by a length table; this call
 * serves both parts from the shared blocks in one launch:
 *   request r holds L = seq_lens[r] resident tokens (its new tokens already
 *   appended, e.g. by bkv_kv_append; reading Q7) and its LAST
 *   n = cu_q[r+1] - cu_q[r] tokens are queries.  Query i (0 <= i < n) is
 *   logical token p = L - n + i and attends causally:
 *     out[cu_q[r]+i][h] = softmax_{t <= p}(softmax_scale * q . K_r[t]) . V_r[t]
 *   with kv head h / (num_q_heads / num_kv_heads).  n = 1 is decode attention
 *   (same result as bkv_paged_decode_attention up to fp32 summation order);
 *   n = L is full causal prefill; n = 0 leaves the request untouched.
 *   cu_q        device int32 [num_seqs+1], non-decreasing, cu_q[0] = 0, n <= L
 *   max_q_len   host upper bound of n (sizes the grid)
 *   q, out      device bf16, element (row i, head h, dim c) at
 *               q[i*q_stride_tok + h*q_stride_head + c] (same for out),
 *               16-byte aligned, strides multiples of 8 elements
 * Dense or general maps (fills).  fp32 accumulation, bf16 RNE output.  No
 * workspace, no split-K (each 128-row query tile runs in one CTA).  head_dim
 * 128 runs on the tcgen05 tensor cores; with g = num_q_heads / num_kv_heads
 * dividing 128, q rows are read by TMA boxes that may start before a
 * request's first row (earlier rows of q, or zero-fill before row 0) but never
 * extend past its last; requests with n = 0 cost no work in batches of up to
 * 512 requests.
 */
BKV_API bkv_status bkv_paged_prefill_attention(const bkv_kv_pool *pool, const bkv_block_map *map,
                                               const int32_t *seq_lens, const int32_t *cu_q,
                                               int32_t max_q_len, const void *q,
                                               int64_t q_stride_tok, int64_t q_stride_head,
                                               int32_t num_q_heads, float softmax_scale, void *out,
                                               int64_t o_stride_tok, int64_t o_stride_head,
                                               bkv_stream_t stream);

/*
 * bkv_paged_mixed_attention -- the paper's dispatch of a mixed batch
 * ("the concatenated prefill requests followed by the
 * decode requests", a length table, each part routed to its kernel).
 * Requests [0, num_prefill_seqs) are served by bkv_paged_prefill_attention
 * (their query rows: cu_q as there, num_prefill_rows = cu_q[num_prefill_seqs]
 * given on the host); requests [num_prefill_seqs, num_seqs) are decodes with
 * ONE query row each, stored contiguously after the prefill rows (request
 * num_prefill_seqs + j at row num_prefill_rows + j), served by the split-K
 * decode kernel (workspace, flags as bkv_paged_decode_attention_ex).  Same
 * results as one bkv_paged_prefill_attention over the whole batch (up to fp32
 * summation order); two launches on `stream` (three with the split merge).
 * With BKV_FLAG_PDL the decode part is launched as a programmatic dependent
 * of the prefill kernel and runs alongside its tail: it reads nothing the
 * prefill writes (disjoint output rows), and the prefill kernel itself starts
 * in plain stream order, after everything before the call.  In a decode-heavy
 * batch (at least 4 decodes per prefill) whose prefill part has at least 8 work
 * items per SM, the prefill's persistent grid then leaves 24 SMs to the decode
 * part from the start.
 */
BKV_API bkv_status bkv_paged_mixed_attention(const bkv_kv_pool *pool, const bkv_block_map *map,
                                             const int32_t *seq_lens, const int32_t *cu_q,
                                             int32_t num_prefill_seqs, int32_t num_prefill_rows,
                                             int32_t max_q_len, int32_t max_seq_len, const void *q,
                                             int64_t q_stride_tok, int64_t q_stride_head,
                                             int32_t num_q_heads, float softmax_scale, void *out,
                                             int64_t o_stride_tok, int64_t o_stride_head,
                                             void *workspace, size_t workspace_bytes,
                                             uint32_t flags, bkv_stream_t stream);

/* Workspace bytes for bkv_paged_decode_attention on the CURRENT device
 * (depends on the SM count); 0 on error (see bkv_last_error). */
BKV_API size_t bkv_decode_workspace_size(int32_t num_seqs, int32_t num_q_heads, int32_t num_kv_heads,
                                 int32_t head_dim);

/*
 * Host-side layout validator on HOST copies of the map.
 * Returns BKV_OK or BKV_ERR_LAYOUT (BKV_ERR_INVALID_ARGUMENT for null inputs).
 * info[0] = invariant code (1 = I4 range/direction/length, 2 = I1 two live
 * tokens on one slot -- the a3/B8 collision of P:731, 3 = I2 more than one
 * forward or reversed entry on a block), info[1..4] = details
 * (I1: r1, t1, r2, t2; I2: block, dir, r1, r2; I4: r, entry or -1, value).
 */
BKV_API bkv_status bkv_validate_layout_host(const int32_t *block_tables, int32_t bt_stride,
                                    const uint8_t *dirs, int32_t dir_row_stride,
                                    int32_t dir_col_stride, int32_t num_seqs,
                                    const int32_t *seq_lens, int32_t num_blocks,
                                    int32_t block_size, int32_t require_nonempty,
                                    int64_t info[5]);

/*
 * The same validator for a dense OR general map, given as a
 * bkv_block_map whose pointers are HOST pointers.  For a general map, I4 also
 * covers num_entries[r] outside [0, bt_stride] (info = 1, r, -1, value), a
 * fill outside [1, block_size] (info = 1, r, e, fill) and seq_lens[r] != the
 * sum of its fills (info = 1, r, -2, seq_len); I1 and I2 are checked over the
 * num_entries[r] entries with the general token -> slot rule.
 */
BKV_API bkv_status bkv_validate_block_map_host(const bkv_block_map *map, const int32_t *seq_lens,
                                               int32_t num_blocks, int32_t block_size,
                                               int32_t require_nonempty, int64_t info[5]);

/*
 * ------------------------------------------------------------------------
 * Planned decode: the split plan made on the HOST once per step, one kernel
 * launch per layer ("computed on device or host").
 *
 * The host scheduler builds each step's length table before it
 * uploads it, so it can also build the split plan there, once, and every
 * layer of the step reuses it.  The plan cuts the flattened sequence of
 * (request r, kv head h, block e) -- r-major, then h, then e -- into equal
 * contiguous ranges, one per warp of a persistent grid (one CTA per SM);
 * rows cut across warps are merged in shared memory inside the kernel, rows
 * cut across CTAs by a small stream-ordered merge kernel (one combined piece
 * per CTA), in an order fixed by the plan, so results are run-to-run bitwise
 * identical.  The plan
 * depends only on the lengths (and entry counts) and on the device's SM
 * count: identical on every rank of a head-sharded TP group.
 *
 * bkv_decode_plan_bytes -- the plan capacity (bytes) for num_seqs requests,
 *   num_kv_heads local kv heads and block tables of bt_stride entries per
 *   request, on a device with num_sms SMs (0: the CURRENT device).  The layout
 *   depends on nothing else, so one buffer of this size serves every step.
 *   Returns 0 on an invalid argument (see bkv_last_error).
 *
 * bkv_decode_plan -- host only; no CUDA call unless num_sms = 0 (then one
 *   cached query of the current device's SM count).
 *   seq_lens     HOST int32 [num_seqs]: resident lengths the layer calls will
 *                receive (after this step's append), >= 0
 *   map          the step's block map with HOST pointers (block_tables,
 *                dirs, and fills/num_entries for a general map, f3) -- the
 *                plan carries it flattened in warp order, packed per entry
 *                (block id < 2^25, direction, live tokens, last-entry bit),
 *                so the layer kernels read no block table
 *   num_kv_heads, num_q_heads, head_dim, block_size: the layer geometry
 *   num_sms      SM count of the device that will run it (0: current device);
 *                bkv_decode_planned rejects a plan made for another count
 *   plan         HOST buffer, 16-byte aligned, plan_bytes long, written
 *   *plan_bytes_used (optional) bytes of the plan the step must upload (the
 *                layout is fixed; the used bytes end with the step's entries)
 *   The caller copies plan[0, *plan_bytes_used) to a device buffer of
 *   bkv_decode_plan_bytes (one H2D with the step's other metadata) and passes
 *   both copies to every layer.  Fixed layout: a CUDA graph captured with one
 *   step's plan replays any later plan of the same geometry copied into the
 *   same device buffer.
 *   Errors: BKV_ERR_INVALID_ARGUMENT (negative length, entries > bt_stride, a
 *   block id >= 2^25, a direction not 0/1, a fill outside [1, block_size] or
 *   fills not summing to the length, problem >= 2^30 blocks x heads),
 *   BKV_ERR_UNSUPPORTED (geometry outside the built set),
 *   BKV_ERR_WORKSPACE_TOO_SMALL (plan_bytes below the capacity).
 *
 * bkv_decode_planned -- one layer: decode attention (k_new = v_new = NULL,
 *   semantics of bkv_paged_decode_attention_ex) or the fused decode step
 *   (both set, semantics of bkv_decode_step), with optional peer outputs
 *   (semantics of bkv_decode_multi_out; n_peers = 0, peer_outs = NULL for
 *   none).  Two launches (the decode kernel and the cross-CTA merge kernel).
 *   plan_host    the buffer bkv_decode_plan wrote (only its header is read)
 *   plan_dev     device copy of it, 16-byte aligned
 *   map          the step's block map (device pointers): the plan already holds
 *                it flattened; read by the dynamically scheduled path below
 *   seq_lens     device int32 [num_seqs], the lengths the plan was built from
 *   workspace    as bkv_paged_decode_attention (bkv_decode_workspace_size;
 *                zero-initialised once: the kernel leaves its counters zero)
 *   flags        BKV_FLAG_PDL (| BKV_FLAG_KV_EARLY): programmatic dependent launch; the plan,
 *                seq_lens and the block map (block_tables, dirs, fills,
 *                num_entries) are read BEFORE the preceding kernel on the
 *                stream completes, so none of them may be written by that
 *                kernel (host copies and earlier kernels are fine); q, k_new,
 *                v_new, the pool and the workspace are read after it.
 *   Large problems (plan ranges of >= 128 blocks per warp, e.g. OPT-30B on one
 *   GPU) run the dynamically scheduled kernel pair of bkv_decode_multi_out
 *   instead (same results up to fp32 summation order): over a long kernel the
 *   per-SM bandwidth spread outweighs the static plan's savings.
 *   Errors: as bkv_decode_multi_out, plus BKV_ERR_INVALID_ARGUMENT when the
 *   plan's geometry (num_seqs, heads, group, head_dim, block_size, dense or
 *   general map, SM count) does not match the call.
 */
BKV_API size_t bkv_decode_plan_bytes(int32_t num_seqs, int32_t num_kv_heads, int32_t bt_stride,
                                     int32_t num_sms);
BKV_API bkv_status bkv_decode_plan(const int32_t *seq_lens, const bkv_block_map *map, int32_t num_kv_heads,
                                   int32_t num_q_heads, int32_t head_dim, int32_t block_size, int32_t num_sms,
                                   void *plan, size_t plan_bytes, size_t *plan_bytes_used);
BKV_API bkv_status bkv_decode_planned(const bkv_kv_pool *pool, const bkv_block_map *map,
                                      const int32_t *seq_lens, const void *plan_host, const void *plan_dev,
                                      const void *k_new, const void *v_new, const void *q,
                                      int64_t q_stride_seq, int64_t q_stride_head, int32_t num_q_heads,
                                      float softmax_scale, void *out, int64_t o_stride_seq,
                                      int64_t o_stride_head, void *const *peer_outs, int32_t n_peers,
                                      void *workspace, size_t workspace_bytes, uint32_t flags,
                                      bkv_stream_t stream);

/* Developer switches (BKV_* environment variables) are read once
 * per process; this re-reads them (tests and A/B runs; not concurrent-safe). */
BKV_API void bkv_reload_dev_switches(void);

BKV_API const char *bkv_status_string(bkv_status s);
BKV_API const char *bkv_last_error(void); /* thread-local detail of the last failure */
BKV_API int32_t bkv_version(void);        /* MAJOR*10000 + MINOR*100 + PATCH (0.3.0: planned decode) */

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* BKV_H_ */
