// decode_plan.cu -- host-side static split plan for the planned decode kernel
// ("Per (r, kv_head): block-aligned splits ... computed on
// device or host"; DESIGN.md §6 "planned decode").
//
// The host scheduler already holds every request's length when it builds the
// step's block tables (PAPER.md: the length table the kernel reads),
// so the split plan is made there once per step and reused by all layers:
//
//   * The flattened sequence of (request r, kv head h, block e) -- r-major,
//     then h, then e -- holds N = H * sum_r nb_r blocks.  Warp w of the
//     persistent grid (grid = SM count, kPlannedWarps warps per CTA) streams
//     the contiguous range [w P, (w+1) P), P = ceil(N / W): every warp moves
//     the same number of bytes, so the step is not bounded by the longest
//     request (the small-shard regime of Llama-2-70B TP8).
//   * A range cut at row boundaries gives the warp's segments.  A row wholly
//     inside one warp is written by that warp; a row cut across warps leaves
//     a piece (m, l, o) in the warp's shared memory, and the CTA combines the
//     pieces of its warps after its last block (merge task, mode 0).  A row
//     cut across CTAs has one combined piece per CTA in the workspace; the
//     last CTA to arrive combines them in CTA order (mode 1).  The combine
//     order is fixed by the plan, so results are run-to-run deterministic.
//   * The step's block map travels inside the plan, flattened in the same order
//     and packed (block id, direction, live tokens, last-entry bit): a warp's
//     blocks are a contiguous slice of that list, so the kernel reads no block
//     table and its first tile needs one dependent load.
//   * Rows with no tokens (reading Q8) get zeros.
//   * The layout has fixed capacities (offsets depend on num_seqs, kv heads and
//     the grid only), so a captured CUDA graph replays any later plan of the
//     same geometry copied into the same device buffer; the kernels read the
//     per-step counts from the device copy of the header.
#include <string.h>

#include <algorithm>
#include <vector>

#include "../../include/bkv.h"
#include "bkv_internal.h"

namespace bkv {

namespace {
size_t up4(size_t x) { return (x + 3) & ~size_t(3); }

// Fixed-capacity layout: the array offsets depend only on (B, H, grid, warps), never on
// the lengths, so a CUDA graph captured with one step's plan stays valid when the next
// step's plan (same geometry) is copied into the same device buffer.
struct PlanLayout {
  size_t off_wseg, off_segs, off_ctask, off_tasks, off_zero, off_xrows, off_ent, words;
  size_t cap_segs, cap_tasks, cap_zero, cap_xrows, cap_ent;
};
PlanLayout plan_layout(int B, int H, int bt_stride, int grid, int warps) {
  const size_t W = static_cast<size_t>(grid) * warps, BH = static_cast<size_t>(B) * H;
  PlanLayout l;
  l.cap_segs = W + BH;        // each warp range starts one segment, each row start another
  l.cap_tasks = 2 * W;        // a warp has at most two split segments, one task each
  l.cap_zero = BH;
  l.cap_xrows = grid;         // each CTA boundary cuts at most one row
  l.off_wseg = sizeof(PlanHeader) / 4;
  l.off_segs = up4(l.off_wseg + W + 1);
  l.off_ctask = up4(l.off_segs + 8 * l.cap_segs);
  l.off_tasks = up4(l.off_ctask + grid + 1);
  l.off_zero = up4(l.off_tasks + 8 * l.cap_tasks);
  l.off_xrows = up4(l.off_zero + 2 * l.cap_zero);
  l.cap_ent = BH * static_cast<size_t>(bt_stride);   // last: the bytes a step uploads end with its entries
  l.off_ent = up4(l.off_xrows + 4 * l.cap_xrows);
  l.words = up4(l.off_ent + l.cap_ent);
  return l;
}
}  // namespace

size_t plan_words_bound(int B, int H, int bt_stride, int grid, int warps) {
  return plan_layout(B, H, bt_stride, grid, warps).words;
}

// Returns 0 on success, else a message (static string) for the caller's fail().
const char *build_plan(const int32_t *seq_lens, const HostMap &map, int B, int H, int g, int D, int bs, int grid,
                       int warps, int32_t *out, size_t out_words, size_t *used_words) {
  const int W = grid * warps;
  const int32_t *num_entries = map.fills ? map.nent : nullptr;
  const int max_entries = map.bt_stride;
  std::vector<int64_t> pre(B + 1, 0);
  for (int r = 0; r < B; ++r) {
    const int32_t L = seq_lens[r];
    if (L < 0) return "seq_lens[r] < 0";
    int64_t nb;
    if (num_entries) {
      nb = num_entries[r];
      if (nb < 0) return "num_entries[r] < 0";
      if ((nb == 0) != (L == 0)) return "num_entries[r] and seq_lens[r] disagree on an empty request";
    } else {
      nb = (static_cast<int64_t>(L) + bs - 1) / bs;
    }
    if (nb > max_entries) return "a request needs more block-table entries than bt_stride";
    pre[r + 1] = pre[r] + nb;
  }
  const int64_t N64 = pre[B] * H;
  if (N64 >= (int64_t(1) << 30)) return "problem too large for one plan (blocks x heads >= 2^30)";
  const int N = static_cast<int>(N64);
  const int P = std::max(1, (N + W - 1) / W);

  struct Seg { int r, h, e0, e1, split; };
  std::vector<std::vector<Seg>> wsegs(W);
  std::vector<std::vector<PlanTask>> ctasks(grid);
  std::vector<int32_t> zero, xrows;
  int max_pieces = 1;
  for (int r = 0; r < B; ++r) {
    const int nb = static_cast<int>(pre[r + 1] - pre[r]);
    for (int h = 0; h < H; ++h) {
      if (nb == 0) {
        zero.push_back(r);
        zero.push_back(h);
        continue;
      }
      const int base = static_cast<int>(H * pre[r]) + h * nb;
      const int w0 = base / P, w1 = (base + nb - 1) / P;
      const int split = w1 > w0 ? 1 : 0;
      // slot of warp w0's piece: 0 when it is the warp's first segment
      const int wa_slot_row = wsegs[w0].empty() ? 0 : 1;
      for (int w = w0; w <= w1; ++w) {
        const int lo = std::max(base, w * P), hi = std::min(base + nb, (w + 1) * P);
        wsegs[w].push_back(Seg{r, h, lo - base, hi - base, split});
      }
      if (!split) continue;
      const int c0 = w0 / warps, c1 = w1 / warps, n = c1 - c0 + 1;
      max_pieces = std::max(max_pieces, n);
      const int flag0 = (base == c0 * warps * P) ? 0 : 1;
      if (n > 1) {
        xrows.push_back(r);
        xrows.push_back(h);
        xrows.push_back(c0);
        xrows.push_back(n | (flag0 << 16));
      }
      for (int c = c0; c <= c1; ++c) {
        PlanTask t;
        const int wa = std::max(w0, c * warps) - c * warps, wb = std::min(w1, c * warps + warps - 1) - c * warps;
        const int wa_slot = (c == c0) ? wa_slot_row : 0;
        t.r = r;
        t.h = h;
        t.warps = wa | (wb << 8) | (wa_slot << 16);
        t.mode = n > 1 ? 1 : 0;
        t.c0 = c0;
        t.n = n;
        t.flag0 = flag0;
        t.gslot = (c == c0) ? 2 * c0 + flag0 : 2 * c;
        ctasks[c].push_back(t);
      }
    }
  }
  size_t n_segs = 0, n_tasks = 0;
  for (auto &v : wsegs) n_segs += v.size();
  for (auto &v : ctasks) n_tasks += v.size();
  const PlanLayout lay = plan_layout(B, H, max_entries, grid, warps);
  if (n_segs > lay.cap_segs || n_tasks > lay.cap_tasks || zero.size() / 2 > lay.cap_zero ||
      xrows.size() / 4 > lay.cap_xrows)
    return "internal: plan exceeds its fixed capacity";
  const size_t off_wseg = lay.off_wseg, off_segs = lay.off_segs, off_ctask = lay.off_ctask;
  const size_t off_tasks = lay.off_tasks, off_zero = lay.off_zero, off_xrows = lay.off_xrows;
  const size_t off_ent = lay.off_ent;
  const size_t words = off_ent + static_cast<size_t>(N);   // used bytes (the capacity is lay.words)
  *used_words = words;
  if (lay.words > out_words) return "plan buffer too small";
  if (lay.words >= (size_t(1) << 31)) return "plan too large";
  // the step's entries in flattened (r, h, e) order, packed: block | dir << 25 | (n - 1) << 26 | last << 31
  // (dense map: every entry but the last holds bs tokens; general map: the entry's fill, f3)
  std::vector<uint32_t> row_ent;
  uint32_t *ent = reinterpret_cast<uint32_t *>(out + off_ent);
  size_t pos = 0;
  for (int r = 0; r < B; ++r) {
    const int nb = static_cast<int>(pre[r + 1] - pre[r]);
    row_ent.resize(nb);
    int64_t sum = 0;
    for (int e = 0; e < nb; ++e) {
      const int64_t blk = map.bt[static_cast<int64_t>(r) * map.bt_stride + e];
      const int dir = map.dirs[static_cast<int64_t>(r) * map.dir_rs + static_cast<int64_t>(e) * map.dir_cs];
      const int n = map.fills ? map.fills[static_cast<int64_t>(r) * map.fill_rs + e]
                              : static_cast<int>(std::min<int64_t>(bs, seq_lens[r] - static_cast<int64_t>(e) * bs));
      if (blk < 0 || blk > static_cast<int64_t>(kEntBlockMask)) return "a block id is negative or >= 2^25";
      if (dir < 0 || dir > 1) return "a direction flag is not 0 or 1";
      if (n < 1 || n > bs) return "an entry holds no token or more than block_size (fills)";
      sum += n;
      row_ent[e] = static_cast<uint32_t>(blk) | (static_cast<uint32_t>(dir) << kEntDirShift) |
                   (static_cast<uint32_t>(n - 1) << kEntFillShift) | (e == nb - 1 ? 1u << kEntLastShift : 0u);
    }
    if (map.fills && sum != seq_lens[r]) return "seq_lens[r] differs from the sum of its fills";
    for (int h = 0; h < H; ++h)
      for (int e = 0; e < nb; ++e) ent[pos++] = row_ent[e];
  }
  memset(out, 0, off_ent * 4);
  PlanHeader *hd = reinterpret_cast<PlanHeader *>(out);
  hd->magic = kPlanMagic;
  hd->version = kPlanVersion;
  hd->words = static_cast<int32_t>(words);
  hd->B = B;
  hd->H = H;
  hd->g = g;
  hd->D = D;
  hd->bs = bs;
  hd->general = num_entries ? 1 : 0;
  hd->grid = grid;
  hd->warps = warps;
  hd->P = P;
  hd->n_segs = static_cast<int32_t>(n_segs);
  hd->n_tasks = static_cast<int32_t>(n_tasks);
  hd->n_zero = static_cast<int32_t>(zero.size() / 2);
  hd->total = N;
  hd->off_wseg = static_cast<int32_t>(off_wseg);
  hd->off_segs = static_cast<int32_t>(off_segs);
  hd->off_ctask = static_cast<int32_t>(off_ctask);
  hd->off_tasks = static_cast<int32_t>(off_tasks);
  hd->off_zero = static_cast<int32_t>(off_zero);
  hd->max_pieces = max_pieces;
  hd->max_entries = max_entries;
  hd->off_xrows = static_cast<int32_t>(off_xrows);
  hd->n_xrows = static_cast<int32_t>(xrows.size() / 4);
  hd->off_ent = static_cast<int32_t>(off_ent);
  hd->n_ent = N;
  int32_t *wseg = out + off_wseg, *segs = out + off_segs, *ctask = out + off_ctask, *tasks = out + off_tasks;
  size_t k = 0;
  for (int w = 0; w < W; ++w) {
    wseg[w] = static_cast<int32_t>(k);
    for (const Seg &s : wsegs[w]) {
      segs[8 * k + 0] = s.r;
      segs[8 * k + 1] = s.h;
      segs[8 * k + 2] = s.e0;
      segs[8 * k + 3] = s.e1 | (s.split << kPlanSplitBit);
      segs[8 * k + 4] = seq_lens[s.r];                                // L of the row (informational)
      segs[8 * k + 5] = static_cast<int32_t>(pre[s.r + 1] - pre[s.r]); // its entries
      ++k;
    }
  }
  wseg[W] = static_cast<int32_t>(k);
  k = 0;
  for (int c = 0; c < grid; ++c) {
    if (ctasks[c].size() > static_cast<size_t>(2 * warps)) return "internal: more than 2 merge tasks per warp";
    ctask[c] = static_cast<int32_t>(k);
    for (const PlanTask &t : ctasks[c]) memcpy(tasks + 8 * k++, &t, sizeof t);
  }
  ctask[grid] = static_cast<int32_t>(k);
  if (!zero.empty()) memcpy(out + off_zero, zero.data(), zero.size() * 4);
  if (!xrows.empty()) memcpy(out + off_xrows, xrows.data(), xrows.size() * 4);
  return nullptr;
}

}  // namespace bkv
