/*
 * bkv_oracle.c -- CPU reference for BROS bidirectional paged decode attention.
 *
 * TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct C (fp64 where
 * floating point is involved).  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_2504_09590_b200/csrc); the product never links or calls it.
 *
 * Citations: "P:NNN" = line NNN of PAPER.md (arXiv 2504.09590, the BROS paper);
 * readings Q1..Q16 are listed in DESIGN.md "Readings of the paper".
 *
 * Pinning: slot map -> golden fixtures of P:711 and
 * the a3/B8 collision rule of P:731; append/gather -> identity on random
 * layouts + flat-array stress; attention -> closed forms (L=1, equal keys,
 * scale 0, equal values, dominant key) and torch SDPA in float64 on dense
 * arrays; validator -> hand-built violating layouts.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* bf16 -> double: the bf16 bit pattern is the top half of an IEEE float32 (exact). */
static double bf16_to_f64(uint16_t b) {
    uint32_t u = ((uint32_t)b) << 16;
    float f;
    memcpy(&f, &u, sizeof f);
    return (double)f;
}

double bkvo_bf16_to_f64(uint16_t b) { return bf16_to_f64(b); }

/*
 * Slot of the j-th token of a block (§5.1 "Block Structure"):
 * "KV cache of the RT request occupies memory slots from the left to the right
 * in the block while that of the BE request in the opposite direction".
 * Direction flag: 0 = RT, left->right; 1 = BE, right->left
 * ("whenever the flag of direction is evaluated to be true" -> invert).
 * Reading Q3: the reversed j-th slot is bs-1-j.
 */
int bkvo_slot_in_block(int dir, int64_t t, int bs) {
    int j = (int)(t % bs);
    return dir ? (bs - 1 - j) : j;
}

static uint8_t dir_of(const uint8_t *dirs, int rs, int cs, int r, int e) {
    return dirs[(int64_t)r * rs + (int64_t)e * cs];
}

/*
 * Logical token t of request r -> (physical block, slot), the block map of
 * block-table entry e = t div bs.
 */
static void locate(const int32_t *bt, int bt_stride, const uint8_t *dirs, int rs, int cs,
                   int bs, int r, int64_t t, int32_t *blk, int *slot) {
    int64_t e = t / bs;
    *blk = bt[(int64_t)r * bt_stride + e];
    *slot = bkvo_slot_in_block(dir_of(dirs, rs, cs, r, (int)e), t, bs);
}

/*
 * Layout validator.  Returns
 *   0 ok
 *   1 I4: block id out of range / direction not in {0,1} / length out of range
 *   2 I1: two live tokens map to the same (block, slot)  -- the a3/B8 collision
 *   3 I2: a physical block referenced by more than one forward or more than one
 *         reversed block-table entry ("one RT request and one BE request")
 * info[0..3] describes the first violation: I1 -> (r1, t1, r2, t2); I2 -> (block, dir, r1, r2);
 * I4 -> (r, e or -1, value, 0).
 * Because lengths include this step's appended tokens (reading Q7), I1 over
 * the post-append lengths is also I5 (appended slots disjoint from each other
 * and from every live token).
 */
int bkvo_validate(int B, const int32_t *bt, int bt_stride, const uint8_t *dirs, int rs, int cs,
                  const int32_t *lens, int num_blocks, int bs, int require_nonempty,
                  int64_t *info) {
    for (int k = 0; k < 4; ++k) info[k] = 0;
    for (int r = 0; r < B; ++r) {
        int64_t L = lens[r];
        if (L < 0 || L > (int64_t)bt_stride * bs || (require_nonempty && L < 1)) {
            info[0] = r; info[1] = -1; info[2] = L;
            return 1;
        }
        int64_t nb = (L + bs - 1) / bs;
        for (int64_t e = 0; e < nb; ++e) {
            int32_t b = bt[(int64_t)r * bt_stride + e];
            uint8_t d = dir_of(dirs, rs, cs, r, (int)e);
            if (b < 0 || b >= num_blocks) { info[0] = r; info[1] = e; info[2] = b; return 1; }
            if (d > 1) { info[0] = r; info[1] = e; info[2] = d; return 1; }
        }
    }
    /* I2: count forward and reversed entries per physical block */
    int32_t *fwd_owner = malloc(sizeof(int32_t) * (size_t)num_blocks);
    int32_t *rev_owner = malloc(sizeof(int32_t) * (size_t)num_blocks);
    for (int b = 0; b < num_blocks; ++b) fwd_owner[b] = rev_owner[b] = -1;
    int rc = 0;
    for (int r = 0; r < B && !rc; ++r) {
        int64_t nb = (lens[r] + bs - 1) / bs;
        for (int64_t e = 0; e < nb; ++e) {
            int32_t b = bt[(int64_t)r * bt_stride + e];
            uint8_t d = dir_of(dirs, rs, cs, r, (int)e);
            int32_t *own = d ? rev_owner : fwd_owner;
            if (own[b] >= 0) { info[0] = b; info[1] = d; info[2] = own[b]; info[3] = r; rc = 3; break; }
            own[b] = r;
        }
    }
    free(fwd_owner); free(rev_owner);
    if (rc) return rc;
    /* I1: every live (r, t) occupies a distinct (block, slot) */
    int64_t nslots = (int64_t)num_blocks * bs;
    int32_t *who_r = malloc(sizeof(int32_t) * (size_t)nslots);
    int64_t *who_t = malloc(sizeof(int64_t) * (size_t)nslots);
    for (int64_t s = 0; s < nslots; ++s) who_r[s] = -1;
    for (int r = 0; r < B && !rc; ++r) {
        for (int64_t t = 0; t < lens[r]; ++t) {
            int32_t blk; int slot;
            locate(bt, bt_stride, dirs, rs, cs, bs, r, t, &blk, &slot);
            int64_t s = (int64_t)blk * bs + slot;
            if (who_r[s] >= 0) {
                info[0] = who_r[s]; info[1] = who_t[s]; info[2] = r; info[3] = t;
                rc = 2; break;
            }
            who_r[s] = r; who_t[s] = t;
        }
    }
    free(who_r); free(who_t);
    return rc;
}

/*
 * kv_append (P:711 write rule): for request r and its
 * j-th new token (logical position t = before[r] + j) copy the K and V rows of
 * every head into that token's slot.  Pure copy, nothing else changes.
 * Pool element (block, head, slot, i) lives at block*sb + head*sh + slot*ss + i.
 * slot_mapping_out (optional) receives block*bs + slot per new token.
 */
void bkvo_append(uint16_t *K, uint16_t *V, int64_t sb, int64_t sh, int64_t ss,
                 int H, int d, int bs,
                 int B, const int32_t *bt, int bt_stride, const uint8_t *dirs, int rs, int cs,
                 const int32_t *before, const int32_t *cu_new,
                 const uint16_t *k_new, const uint16_t *v_new, int64_t *slot_mapping_out) {
    for (int r = 0; r < B; ++r) {
        for (int32_t i = cu_new[r]; i < cu_new[r + 1]; ++i) {
            int64_t t = (int64_t)before[r] + (i - cu_new[r]);
            int32_t blk; int slot;
            locate(bt, bt_stride, dirs, rs, cs, bs, r, t, &blk, &slot);
            for (int h = 0; h < H; ++h) {
                int64_t dst = (int64_t)blk * sb + (int64_t)h * sh + (int64_t)slot * ss;
                int64_t src = ((int64_t)i * H + h) * d;
                memcpy(K + dst, k_new + src, sizeof(uint16_t) * (size_t)d);
                memcpy(V + dst, v_new + src, sizeof(uint16_t) * (size_t)d);
            }
            if (slot_mapping_out) slot_mapping_out[i] = (int64_t)blk * bs + slot;
        }
    }
}

/*
 * gather: dense K_r[t][h][:], V_r[t][h][:] for t < L in
 * LOGICAL token order, read back through the bidirectional block table.
 */
void bkvo_gather(const uint16_t *K, const uint16_t *V, int64_t sb, int64_t sh, int64_t ss,
                 int H, int d, int bs,
                 const int32_t *bt, int bt_stride, const uint8_t *dirs, int rs, int cs,
                 int r, int64_t L, uint16_t *k_out, uint16_t *v_out) {
    for (int64_t t = 0; t < L; ++t) {
        int32_t blk; int slot;
        locate(bt, bt_stride, dirs, rs, cs, bs, r, t, &blk, &slot);
        for (int h = 0; h < H; ++h) {
            int64_t src = (int64_t)blk * sb + (int64_t)h * sh + (int64_t)slot * ss;
            memcpy(k_out + (t * H + h) * d, K + src, sizeof(uint16_t) * (size_t)d);
            memcpy(v_out + (t * H + h) * d, V + src, sizeof(uint16_t) * (size_t)d);
        }
    }
}

/*
 * Decode attention, exact in fp64 (the cost model's
 * "attention score matrix ... batched general matrix multiplication and
 * softmax").  For query head h of request r with kv head
 * kv = h / g (reading Q9, g = Hq / H):
 *   s_t = scale * sum_i q[h][i] * K_r[t][kv][i]
 *   m   = max_t s_t,  p_t = exp(s_t - m)
 *   o   = sum_t p_t * V_r[t][kv] / sum_t p_t
 * q is bf16 [B][Hq][d] (contiguous), out is fp64 [B][Hq][d].
 * L = 0 gives o = 0 (reading Q8).  Requests in [r_begin, r_end) only.
 */
void bkvo_attention(const uint16_t *K, const uint16_t *V, int64_t sb, int64_t sh, int64_t ss,
                    int H, int d, int bs,
                    const int32_t *bt, int bt_stride, const uint8_t *dirs, int rs, int cs,
                    const int32_t *lens, int r_begin, int r_end,
                    const uint16_t *q, int Hq, double scale, double *out) {
    int g = Hq / H;
#pragma omp parallel for schedule(dynamic, 1)
    for (int r = r_begin; r < r_end; ++r) {
        int64_t L = lens[r];
        double *o_r = out + (int64_t)r * Hq * d;
        if (L <= 0) { memset(o_r, 0, sizeof(double) * (size_t)Hq * d); continue; }
        uint16_t *kr = malloc(sizeof(uint16_t) * (size_t)(L * H * d));
        uint16_t *vr = malloc(sizeof(uint16_t) * (size_t)(L * H * d));
        double *s = malloc(sizeof(double) * (size_t)L);
        bkvo_gather(K, V, sb, sh, ss, H, d, bs, bt, bt_stride, dirs, rs, cs, r, L, kr, vr);
        for (int h = 0; h < Hq; ++h) {
            int kv = h / g;
            const uint16_t *qh = q + ((int64_t)r * Hq + h) * d;
            double m = -INFINITY;
            for (int64_t t = 0; t < L; ++t) {
                const uint16_t *kt = kr + (t * H + kv) * d;
                double acc = 0.0;
                for (int i = 0; i < d; ++i) acc += bf16_to_f64(qh[i]) * bf16_to_f64(kt[i]);
                s[t] = scale * acc;
                if (s[t] > m) m = s[t];
            }
            double denom = 0.0;
            double *oh = o_r + (int64_t)h * d;
            for (int i = 0; i < d; ++i) oh[i] = 0.0;
            for (int64_t t = 0; t < L; ++t) {
                double p = exp(s[t] - m);
                denom += p;
                const uint16_t *vt = vr + (t * H + kv) * d;
                for (int i = 0; i < d; ++i) oh[i] += p * bf16_to_f64(vt[i]);
            }
            for (int i = 0; i < d; ++i) oh[i] /= denom;
        }
        free(kr); free(vr); free(s);
    }
}

/*
 * Lazy checkpointing: copy the K/V rows (every head) of the given
 * physical slots (slot id = block*bs + slot) out of the pool, or back into it
 * on swap-in.  Buffers are [n][H][d].  Pure copies.
 */
void bkvo_checkpoint(const uint16_t *K, const uint16_t *V, int64_t sb, int64_t sh, int64_t ss,
                     int H, int d, int bs, const int64_t *slot_ids, int n,
                     uint16_t *k_out, uint16_t *v_out) {
    for (int i = 0; i < n; ++i) {
        int64_t blk = slot_ids[i] / bs, slot = slot_ids[i] % bs;
        for (int h = 0; h < H; ++h) {
            int64_t src = blk * sb + (int64_t)h * sh + slot * ss;
            memcpy(k_out + ((int64_t)i * H + h) * d, K + src, sizeof(uint16_t) * (size_t)d);
            memcpy(v_out + ((int64_t)i * H + h) * d, V + src, sizeof(uint16_t) * (size_t)d);
        }
    }
}

void bkvo_restore(uint16_t *K, uint16_t *V, int64_t sb, int64_t sh, int64_t ss,
                  int H, int d, int bs, const int64_t *slot_ids, int n,
                  const uint16_t *k_in, const uint16_t *v_in) {
    for (int i = 0; i < n; ++i) {
        int64_t blk = slot_ids[i] / bs, slot = slot_ids[i] % bs;
        for (int h = 0; h < H; ++h) {
            int64_t dst = blk * sb + (int64_t)h * sh + slot * ss;
            memcpy(K + dst, k_in + ((int64_t)i * H + h) * d, sizeof(uint16_t) * (size_t)d);
            memcpy(V + dst, v_in + ((int64_t)i * H + h) * d, sizeof(uint16_t) * (size_t)d);
        }
    }
}

/*
 * Peer slots an append would overwrite (the lazy-checkpoint trigger of
 * P:726-728): for every new token of every request, if its target slot holds
 * a live token of ANOTHER request (per the current lengths `live_lens`),
 * report that victim (request, token, slot id).  Returns the number found
 * (at most cap are written).  O(sum of lengths) with a per-slot owner table.
 */
int bkvo_overwritten_peers(int B, const int32_t *bt, int bt_stride, const uint8_t *dirs, int rs, int cs,
                           const int32_t *live_lens, const int32_t *before, const int32_t *n_new,
                           int num_blocks, int bs, int32_t *victim_r, int64_t *victim_t,
                           int64_t *victim_slot, int cap) {
    int64_t nslots = (int64_t)num_blocks * bs;
    int32_t *own_r = malloc(sizeof(int32_t) * (size_t)nslots);
    int64_t *own_t = malloc(sizeof(int64_t) * (size_t)nslots);
    for (int64_t s = 0; s < nslots; ++s) own_r[s] = -1;
    for (int r = 0; r < B; ++r)
        for (int64_t t = 0; t < live_lens[r]; ++t) {
            int32_t blk; int slot;
            locate(bt, bt_stride, dirs, rs, cs, bs, r, t, &blk, &slot);
            own_r[(int64_t)blk * bs + slot] = r;
            own_t[(int64_t)blk * bs + slot] = t;
        }
    int found = 0;
    for (int r = 0; r < B; ++r)
        for (int32_t j = 0; j < n_new[r]; ++j) {
            int64_t t = (int64_t)before[r] + j;
            int32_t blk; int slot;
            locate(bt, bt_stride, dirs, rs, cs, bs, r, t, &blk, &slot);
            int64_t sid = (int64_t)blk * bs + slot;
            if (own_r[sid] >= 0 && own_r[sid] != r) {
                if (found < cap) {
                    victim_r[found] = own_r[sid];
                    victim_t[found] = own_t[sid];
                    victim_slot[found] = sid;
                }
                ++found;
            }
        }
    free(own_r); free(own_t);
    return found;
}

/*
 * ---------------------------------------------------------------------------
 * General block map (reading Q6 option B).
 *
 * FindBlock places a BE prefill "according to the maximum number of empty
 * slots" and FindPreemptBlock lets an RT request "write its KV cache
 * from the opposite end" of a BE block, so any block -- not just a
 * request's last -- may hold fewer than bs of the request's tokens.  The
 * general map therefore carries, per block-table entry, the number of the
 * request's tokens in it:
 *     fills[r*frs + e] in 1..bs for e < nent[r]
 * Tokens are numbered in entry order: entry e holds tokens
 * [F_e, F_e + fills[e]) with F_e = fills[0] + ... + fills[e-1], and the j-th
 * token of an entry sits at slot j (forward, RT) or bs-1-j (reversed, BE),
 * exactly the in-block rule of P:711.  The request's length is F_{nent[r]}.
 * With every non-last entry full this is the dense map above.
 */
static void locate_f(const int32_t *bt, int bt_stride, const uint8_t *dirs, int rs, int cs,
                     const uint8_t *fills, int frs, int bs, int r, int64_t t,
                     int32_t *blk, int *slot) {
    int64_t e = 0, start = 0;
    while (t >= start + fills[(int64_t)r * frs + e]) {   /* walk the entries in order */
        start += fills[(int64_t)r * frs + e];
        ++e;
    }
    int j = (int)(t - start);                            /* j-th token of entry e */
    *blk = bt[(int64_t)r * bt_stride + e];
    *slot = dir_of(dirs, rs, cs, r, (int)e) ? (bs - 1 - j) : j;
}

/*
 * Validator of a general map: codes as bkvo_validate, plus (code 1, I4)
 * nent[r] outside [0, bt_stride], a fill outside [1, bs] (info = r, e, fill),
 * or lens[r] != sum of the fills (info = r, -1, lens[r], sum).
 */
int bkvo_validate_f(int B, const int32_t *bt, int bt_stride, const uint8_t *dirs, int rs, int cs,
                    const uint8_t *fills, int frs, const int32_t *nent,
                    const int32_t *lens, int num_blocks, int bs, int require_nonempty,
                    int64_t *info) {
    for (int k = 0; k < 4; ++k) info[k] = 0;
    for (int r = 0; r < B; ++r) {
        if (nent[r] < 0 || nent[r] > bt_stride) { info[0] = r; info[1] = -1; info[2] = nent[r]; return 1; }
        int64_t sum = 0;
        for (int e = 0; e < nent[r]; ++e) {
            int f = fills[(int64_t)r * frs + e];
            int32_t b = bt[(int64_t)r * bt_stride + e];
            uint8_t d = dir_of(dirs, rs, cs, r, e);
            if (f < 1 || f > bs) { info[0] = r; info[1] = e; info[2] = f; return 1; }
            if (b < 0 || b >= num_blocks) { info[0] = r; info[1] = e; info[2] = b; return 1; }
            if (d > 1) { info[0] = r; info[1] = e; info[2] = d; return 1; }
            sum += f;
        }
        if (sum != lens[r] || (require_nonempty && lens[r] < 1)) {
            info[0] = r; info[1] = -1; info[2] = lens[r]; info[3] = sum;
            return 1;
        }
    }
    int32_t *fwd_owner = malloc(sizeof(int32_t) * (size_t)num_blocks);
    int32_t *rev_owner = malloc(sizeof(int32_t) * (size_t)num_blocks);
    for (int b = 0; b < num_blocks; ++b) fwd_owner[b] = rev_owner[b] = -1;
    int rc = 0;
    for (int r = 0; r < B && !rc; ++r) {
        for (int e = 0; e < nent[r]; ++e) {
            int32_t b = bt[(int64_t)r * bt_stride + e];
            uint8_t d = dir_of(dirs, rs, cs, r, e);
            int32_t *own = d ? rev_owner : fwd_owner;
            if (own[b] >= 0) { info[0] = b; info[1] = d; info[2] = own[b]; info[3] = r; rc = 3; break; }
            own[b] = r;
        }
    }
    free(fwd_owner); free(rev_owner);
    if (rc) return rc;
    int64_t nslots = (int64_t)num_blocks * bs;
    int32_t *who_r = malloc(sizeof(int32_t) * (size_t)nslots);
    int64_t *who_t = malloc(sizeof(int64_t) * (size_t)nslots);
    for (int64_t s = 0; s < nslots; ++s) who_r[s] = -1;
    for (int r = 0; r < B && !rc; ++r) {
        for (int64_t t = 0; t < lens[r]; ++t) {
            int32_t blk; int slot;
            locate_f(bt, bt_stride, dirs, rs, cs, fills, frs, bs, r, t, &blk, &slot);
            int64_t s = (int64_t)blk * bs + slot;
            if (who_r[s] >= 0) {
                info[0] = who_r[s]; info[1] = who_t[s]; info[2] = r; info[3] = t;
                rc = 2; break;
            }
            who_r[s] = r; who_t[s] = t;
        }
    }
    free(who_r); free(who_t);
    return rc;
}

/* kv_append through a general map (same rule as bkvo_append, token located by locate_f). */
void bkvo_append_f(uint16_t *K, uint16_t *V, int64_t sb, int64_t sh, int64_t ss,
                   int H, int d, int bs,
                   int B, const int32_t *bt, int bt_stride, const uint8_t *dirs, int rs, int cs,
                   const uint8_t *fills, int frs,
                   const int32_t *before, const int32_t *cu_new,
                   const uint16_t *k_new, const uint16_t *v_new, int64_t *slot_mapping_out) {
    for (int r = 0; r < B; ++r) {
        for (int32_t i = cu_new[r]; i < cu_new[r + 1]; ++i) {
            int64_t t = (int64_t)before[r] + (i - cu_new[r]);
            int32_t blk; int slot;
            locate_f(bt, bt_stride, dirs, rs, cs, fills, frs, bs, r, t, &blk, &slot);
            for (int h = 0; h < H; ++h) {
                int64_t dst = (int64_t)blk * sb + (int64_t)h * sh + (int64_t)slot * ss;
                int64_t src = ((int64_t)i * H + h) * d;
                memcpy(K + dst, k_new + src, sizeof(uint16_t) * (size_t)d);
                memcpy(V + dst, v_new + src, sizeof(uint16_t) * (size_t)d);
            }
            if (slot_mapping_out) slot_mapping_out[i] = (int64_t)blk * bs + slot;
        }
    }
}

/* gather through a general map: dense logical-order K_r, V_r for t < L. */
void bkvo_gather_f(const uint16_t *K, const uint16_t *V, int64_t sb, int64_t sh, int64_t ss,
                   int H, int d, int bs,
                   const int32_t *bt, int bt_stride, const uint8_t *dirs, int rs, int cs,
                   const uint8_t *fills, int frs,
                   int r, int64_t L, uint16_t *k_out, uint16_t *v_out) {
    for (int64_t t = 0; t < L; ++t) {
        int32_t blk; int slot;
        locate_f(bt, bt_stride, dirs, rs, cs, fills, frs, bs, r, t, &blk, &slot);
        for (int h = 0; h < H; ++h) {
            int64_t src = (int64_t)blk * sb + (int64_t)h * sh + (int64_t)slot * ss;
            memcpy(k_out + (t * H + h) * d, K + src, sizeof(uint16_t) * (size_t)d);
            memcpy(v_out + (t * H + h) * d, V + src, sizeof(uint16_t) * (size_t)d);
        }
    }
}

/*
 * Decode attention through a general map: gather_f, then exactly the fp64
 * softmax attention of bkvo_attention (readings Q8, Q9).
 */
void bkvo_attention_f(const uint16_t *K, const uint16_t *V, int64_t sb, int64_t sh, int64_t ss,
                      int H, int d, int bs,
                      const int32_t *bt, int bt_stride, const uint8_t *dirs, int rs, int cs,
                      const uint8_t *fills, int frs,
                      const int32_t *lens, int r_begin, int r_end,
                      const uint16_t *q, int Hq, double scale, double *out) {
    int g = Hq / H;
#pragma omp parallel for schedule(dynamic, 1)
    for (int r = r_begin; r < r_end; ++r) {
        int64_t L = lens[r];
        double *o_r = out + (int64_t)r * Hq * d;
        if (L <= 0) { memset(o_r, 0, sizeof(double) * (size_t)Hq * d); continue; }
        uint16_t *kr = malloc(sizeof(uint16_t) * (size_t)(L * H * d));
        uint16_t *vr = malloc(sizeof(uint16_t) * (size_t)(L * H * d));
        double *s = malloc(sizeof(double) * (size_t)L);
        bkvo_gather_f(K, V, sb, sh, ss, H, d, bs, bt, bt_stride, dirs, rs, cs, fills, frs, r, L, kr, vr);
        for (int h = 0; h < Hq; ++h) {
            int kv = h / g;
            const uint16_t *qh = q + ((int64_t)r * Hq + h) * d;
            double m = -INFINITY;
            for (int64_t t = 0; t < L; ++t) {
                const uint16_t *kt = kr + (t * H + kv) * d;
                double acc = 0.0;
                for (int i = 0; i < d; ++i) acc += bf16_to_f64(qh[i]) * bf16_to_f64(kt[i]);
                s[t] = scale * acc;
                if (s[t] > m) m = s[t];
            }
            double denom = 0.0;
            double *oh = o_r + (int64_t)h * d;
            for (int i = 0; i < d; ++i) oh[i] = 0.0;
            for (int64_t t = 0; t < L; ++t) {
                double p = exp(s[t] - m);
                denom += p;
                const uint16_t *vt = vr + (t * H + kv) * d;
                for (int i = 0; i < d; ++i) oh[i] += p * bf16_to_f64(vt[i]);
            }
            for (int i = 0; i < d; ++i) oh[i] /= denom;
        }
        free(kr); free(vr); free(s);
    }
}

/*
 * ---------------------------------------------------------------------------
 * Mixed prefill + decode attention over the bidirectional paged cache
 * (SURVEY §8(f) row f4).  BROS batches "the concatenated prefill requests
 * followed by the decode requests" with a length table and dispatches each
 * part to its attention kernel; the prefill part is standard
 * causal self-attention over the request's tokens (the cost model's
 * "attention score matrix ... batched GEMM and softmax").
 *
 * Request r has L = lens[r] resident tokens (its new tokens already appended,
 * reading Q7); its LAST n = cu_q[r+1] - cu_q[r] tokens are queries.  Query i
 * (0 <= i < n) is logical token p = L - n + i and attends causally to tokens
 * t <= p:
 *   s_t = scale * q_i[h] . K_r[t][kv],  o = sum_{t<=p} e^{s_t - m} V_r[t][kv] / sum_{t<=p} e^{s_t - m}
 * with kv = h / g (reading Q9).  n = 1 is exactly decode attention.
 * q is bf16 [total_q][Hq][d] (row cu_q[r] + i), out fp64 of the same shape.
 * fills == NULL selects the dense map, else the general map (row f3).
 */
void bkvo_prefill_attention(const uint16_t *K, const uint16_t *V, int64_t sb, int64_t sh, int64_t ss,
                            int H, int d, int bs,
                            const int32_t *bt, int bt_stride, const uint8_t *dirs, int rs, int cs,
                            const uint8_t *fills, int frs,
                            int B, const int32_t *lens, const int32_t *cu_q,
                            const uint16_t *q, int Hq, double scale, double *out) {
    int g = Hq / H;
#pragma omp parallel for schedule(dynamic, 1)
    for (int r = 0; r < B; ++r) {
        int64_t L = lens[r];
        int n = cu_q[r + 1] - cu_q[r];
        if (n <= 0) continue;
        uint16_t *kr = malloc(sizeof(uint16_t) * (size_t)(L * H * d));
        uint16_t *vr = malloc(sizeof(uint16_t) * (size_t)(L * H * d));
        double *s = malloc(sizeof(double) * (size_t)L);
        if (fills)
            bkvo_gather_f(K, V, sb, sh, ss, H, d, bs, bt, bt_stride, dirs, rs, cs, fills, frs, r, L, kr, vr);
        else
            bkvo_gather(K, V, sb, sh, ss, H, d, bs, bt, bt_stride, dirs, rs, cs, r, L, kr, vr);
        for (int i = 0; i < n; ++i) {
            int64_t p = L - n + i;                 /* logical position of query i */
            for (int h = 0; h < Hq; ++h) {
                int kv = h / g;
                const uint16_t *qh = q + ((int64_t)(cu_q[r] + i) * Hq + h) * d;
                double *oh = out + ((int64_t)(cu_q[r] + i) * Hq + h) * d;
                double m = -INFINITY;
                for (int64_t t = 0; t <= p; ++t) {
                    const uint16_t *kt = kr + (t * H + kv) * d;
                    double acc = 0.0;
                    for (int c = 0; c < d; ++c) acc += bf16_to_f64(qh[c]) * bf16_to_f64(kt[c]);
                    s[t] = scale * acc;
                    if (s[t] > m) m = s[t];
                }
                double denom = 0.0;
                for (int c = 0; c < d; ++c) oh[c] = 0.0;
                for (int64_t t = 0; t <= p; ++t) {
                    double pt = exp(s[t] - m);
                    denom += pt;
                    const uint16_t *vt = vr + (t * H + kv) * d;
                    for (int c = 0; c < d; ++c) oh[c] += pt * bf16_to_f64(vt[c]);
                }
                for (int c = 0; c < d; ++c) oh[c] /= denom;
            }
        }
        free(kr); free(vr); free(s);
    }
}

int bkvo_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void bkvo_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}
