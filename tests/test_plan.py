"""Host-side split plan of the planned decode (bkv_decode_plan).

CPU only: the plan is built by libbkv's host code for an explicit SM count.
Two kinds of checks:
  * structure -- every (request, kv head, block) of the step lies in exactly one
    warp segment, warp ranges are equal and contiguous, split flags, piece slots,
    merge tasks and global piece slots are consistent and unique;
  * execution -- a float64 numpy model of what the kernel does with the plan
    (per-segment softmax partials, the CTA merge of warp pieces in warp order, the
    cross-CTA merge in CTA order) reproduces plain softmax attention on the dense
    arrays to 1e-12, so the decomposition the plan prescribes is exact.
"""
import numpy as np
import pytest

import paper_2504_09590_b200 as bkv
from synth import make_case

HDR = ("magic", "version", "words", "B", "H", "g", "D", "bs", "general", "grid", "warps", "P",
       "n_segs", "n_tasks", "n_zero", "total", "off_wseg", "off_segs", "off_ctask", "off_tasks",
       "off_zero", "max_pieces", "max_entries", "off_xrows", "n_xrows", "off_ent", "n_ent")


def decode(plan):
    h = {n: int(plan[i]) for i, n in enumerate(HDR)}
    W = h["grid"] * h["warps"]
    wseg = plan[h["off_wseg"]:h["off_wseg"] + W + 1]
    segs8 = plan[h["off_segs"]:h["off_segs"] + 8 * h["n_segs"]].reshape(-1, 8)
    segs = segs8[:, :4]
    ctask = plan[h["off_ctask"]:h["off_ctask"] + h["grid"] + 1]
    tasks = plan[h["off_tasks"]:h["off_tasks"] + 8 * h["n_tasks"]].reshape(-1, 8)
    zero = plan[h["off_zero"]:h["off_zero"] + 2 * h["n_zero"]].reshape(-1, 2)
    return h, wseg, segs, ctask, tasks, zero, segs8[:, 4:6]


def entries(lens, bs, nent):
    return np.asarray(nent if nent is not None else (np.asarray(lens) + bs - 1) // bs, dtype=np.int64)


def check_structure(plan, lens, H, bs, nent=None):
    h, wseg, segs, ctask, tasks, zero, lnb = decode(plan)
    nb = entries(lens, bs, nent)
    assert np.array_equal(lnb[:, 0], np.asarray(lens)[segs[:, 0]]) and np.array_equal(lnb[:, 1], nb[segs[:, 0]])
    B = len(lens)
    W = h["grid"] * h["warps"]
    N = int(nb.sum()) * H
    P = h["P"]
    assert h["total"] == N and P == max(1, -(-N // W))
    assert wseg[0] == 0 and wseg[-1] == len(segs) and np.all(np.diff(wseg) >= 0)
    seen = {}
    pieces = {}                                 # (r, h) -> [(warp, seg index in warp)]
    for w in range(W):
        pos = w * P                             # flattened position the warp's range starts at
        for k, si in enumerate(range(wseg[w], wseg[w + 1])):
            r, hh, e0, w4 = (int(x) for x in segs[si])
            e1, split = w4 & 0xFFFF, (w4 >> 30) & 1
            assert 0 <= r < B and 0 <= hh < H and 0 <= e0 < e1 <= nb[r]
            base = int(H * nb[:r].sum() + hh * nb[r])
            assert base + e0 == pos, "segments of a warp are contiguous in the flattened order"
            pos += e1 - e0
            for e in range(e0, e1):
                assert (r, hh, e) not in seen
                seen[(r, hh, e)] = w
            pieces.setdefault((r, hh), []).append((w, k, split, e0, e1))
        assert pos - w * P <= P and (pos == min(N, (w + 1) * P) or wseg[w + 1] == wseg[w])
    assert len(seen) == N, "every (request, kv head, block) is streamed exactly once"
    # split flags and piece slots: warp w0's piece is slot 0 iff it is the warp's first segment
    for (r, hh), ps in pieces.items():
        ws_ = [p[0] for p in ps]
        assert ws_ == list(range(ws_[0], ws_[-1] + 1))
        assert all(p[2] == (len(ps) > 1) for p in ps)
        assert all(p[1] == 0 for p in ps[1:]), "pieces after the first open their warp's range"
    # zero rows
    zr = {(int(a), int(b)) for a, b in zero}
    assert zr == {(r, hh) for r in range(B) for hh in range(H) if nb[r] == 0}
    # merge tasks: one per (split row, CTA it touches); CTA pieces in global slots
    wc = h["warps"]
    gslots = set()
    got = {}
    for c in range(h["grid"]):
        for t in tasks[ctask[c]:ctask[c + 1]]:
            r, hh, wpk, mode, c0, n, flag0, gslot = (int(x) for x in t)
            wa, wb, wa_slot = wpk & 0xFF, (wpk >> 8) & 0xFF, (wpk >> 16) & 1
            got.setdefault((r, hh), []).append((c, wa, wb, wa_slot, mode, c0, n, flag0, gslot))
            if mode == 1:
                assert gslot not in gslots
                gslots.add(gslot)
                assert gslot == (2 * c0 + flag0 if c == c0 else 2 * c)
    xr = plan[h["off_xrows"]:h["off_xrows"] + 4 * h["n_xrows"]].reshape(-1, 4)
    xset = {(int(a), int(b)): (int(c), int(w) & 0xFFFF, int(w) >> 16) for a, b, c, w in xr}
    assert len(xset) == len(xr)
    cross = {k: (v[0][5], v[0][6], v[0][7]) for k, v in got.items() if v[0][4] == 1}
    assert xset == cross, "xrows lists exactly the rows cut across CTAs"
    for (r, hh), ps in pieces.items():
        if len(ps) == 1:
            assert (r, hh) not in got
            continue
        ts = got[(r, hh)]
        ctas = sorted({p[0] // wc for p in ps})
        assert [t[0] for t in ts] == ctas
        for t in ts:
            c, wa, wb, wa_slot, mode, c0, n, flag0, _ = t
            mine = [p for p in ps if p[0] // wc == c]
            assert (wa, wb) == (mine[0][0] - c * wc, mine[-1][0] - c * wc)
            assert wa_slot == (0 if mine[0][1] == 0 else 1)
            assert (mode, c0, n) == (int(len(ctas) > 1), ctas[0], len(ctas))
    return h


def simulate(plan, lens, H, g, bs, q, K, V, nent=None, fills=None):
    """float64 model of the planned kernel's decomposition (log2-domain softmax pieces)."""
    h, wseg, segs, ctask, tasks, zero, _ = decode(plan)
    B = len(lens)
    W = h["grid"] * h["warps"]
    out = np.full((B, H * g, q.shape[-1]), np.nan)

    def tok_range(r, e):
        if fills is None:
            return e * bs, min(int(lens[r]), (e + 1) * bs)
        f = fills[r][: int(nent[r])].astype(np.int64)
        s = int(f[:e].sum())
        return s, s + int(f[e])

    def piece(r, hh, e0, e1):
        t0, t1 = tok_range(r, e0)[0], tok_range(r, e1 - 1)[1]
        k, v = K[r][t0:t1, hh], V[r][t0:t1, hh]
        s = q[r, hh * g:(hh + 1) * g] @ k.T * np.log2(np.e) / np.sqrt(q.shape[-1])
        m = s.max(1)
        p = np.exp2(s - m[:, None])
        return m, p.sum(1), p @ v

    def merge(ps):
        M = np.max([p[0] for p in ps], axis=0)
        L = sum(p[1] * np.exp2(p[0] - M) for p in ps)
        O = sum(p[2] * np.exp2(p[0] - M)[:, None] for p in ps)
        return M, L, O

    smem = {}
    for w in range(W):
        for k, si in enumerate(range(wseg[w], wseg[w + 1])):
            r, hh, e0, w4 = (int(x) for x in segs[si])
            m, l, o = piece(r, hh, e0, w4 & 0xFFFF)
            if (w4 >> 30) & 1:
                smem[(w, 0 if k == 0 else 1)] = (m, l, o)
            else:
                out[r, hh * g:(hh + 1) * g] = o / l[:, None]
    gp = {}
    finals = []
    for c in range(h["grid"]):
        for t in tasks[ctask[c]:ctask[c + 1]]:
            r, hh, wpk, mode, c0, n, flag0, gslot = (int(x) for x in t)
            wa, wb, wa_slot = wpk & 0xFF, (wpk >> 8) & 0xFF, (wpk >> 16) & 1
            base = c * h["warps"]
            ps = [smem[(base + wa + k, wa_slot if k == 0 else 0)] for k in range(wb - wa + 1)]
            M, L, O = merge(ps)
            if mode == 0:
                out[r, hh * g:(hh + 1) * g] = O / L[:, None]
            else:
                gp[gslot] = (M, L, O)
                finals.append((r, hh, c0, n, flag0))
    for r, hh, c0, n, flag0 in set(finals):
        ps = [gp[2 * c0 + flag0 if k == 0 else 2 * (c0 + k)] for k in range(n)]
        M, L, O = merge(ps)
        out[r, hh * g:(hh + 1) * g] = O / L[:, None]
    for r, hh in zero:
        out[r, hh * g:(hh + 1) * g] = 0.0
    return out


def dense_attention(lens, H, g, q, K, V):
    out = np.zeros_like(q)
    for r in range(len(lens)):
        for hq in range(H * g):
            L = int(lens[r])
            if L == 0:
                continue
            k, v = K[r][:L, hq // g], V[r][:L, hq // g]
            s = k @ q[r, hq] / np.sqrt(q.shape[-1])
            p = np.exp(s - s.max())
            out[r, hq] = p @ v / p.sum()
    return out


def synth_map(lens, bt_stride, seed=0):
    """A block map for bare lengths: distinct random block ids, random per-entry directions."""
    B = len(lens)
    rng = np.random.default_rng(seed)
    ids = rng.permutation(max(1, B * bt_stride)).astype(np.int32)[:B * bt_stride].reshape(B, bt_stride)
    return ids, rng.integers(0, 2, size=(B, bt_stride)).astype(np.uint8)


def _plan(lens, H, g, bs, bt_stride, sms, nent=None, fills=None, d=128, bt=None, dirs=None):
    if bt is None:
        bt, dirs = synth_map(lens, bt_stride)
    return bkv.decode_plan_host(lens, bt, dirs, H, H * g, d, bs, fills=fills, num_entries=nent, num_sms=sms)


def check_entries(plan, lens, H, bs, bt, dirs, nent=None, fills=None):
    """The plan's flattened entry list: every (r, h, e) in flattened order, packed
    block | dir << 25 | (live tokens - 1) << 26 | last << 31."""
    h = decode(plan)[0]
    ent = plan[h["off_ent"]:h["off_ent"] + h["n_ent"]].view(np.uint32)
    nb = entries(lens, bs, nent)
    exp = []
    for r in range(len(lens)):
        row = []
        for e in range(int(nb[r])):
            n = int(fills[r][e]) if fills is not None else min(bs, int(lens[r]) - e * bs)
            dr = int(dirs[r][e]) if np.asarray(dirs).ndim == 2 else int(dirs[r])
            row.append(int(bt[r][e]) | dr << 25 | (n - 1) << 26 | (int(e == nb[r] - 1) << 31))
        exp += row * H
    assert h["n_ent"] == len(exp) and np.array_equal(ent, np.array(exp, dtype=np.uint64).astype(np.uint32))


CASES = [("tiny", 1, 148), ("tiny", 1, 3), ("tiny_gqa", 1, 5), ("opt13b", 8, 148), ("opt13b", 1, 148),
         ("llama70b", 8, 148), ("llama70b", 4, 148), ("llama70b", 1, 148), ("opt30b", 4, 148)]


@pytest.mark.parametrize("cfg,tp,sms", CASES)
def test_plan_structure(cfg, tp, sms):
    case = make_case(cfg, 0)
    sh, lay = case.shape, case.layout
    H = sh.num_kv_heads // tp
    plan = _plan(lay.lens, H, sh.group, sh.block_size, lay.block_tables.shape[1], sms, bt=lay.block_tables,
                 dirs=lay.dirs)
    h = check_structure(plan, lay.lens, H, sh.block_size)
    check_entries(plan, lay.lens, H, sh.block_size, lay.block_tables, lay.dirs)
    assert h["grid"] == sms and h["warps"] == 8


@pytest.mark.parametrize("seed", range(4))
def test_plan_structure_general_and_edge(seed):
    rng = np.random.default_rng(seed)
    case = make_case("tiny_gqa", seed, general=True, share_prob=0.8)
    lay, sh = case.layout, case.shape
    gp = _plan(lay.lens, 2, 4, 16, lay.block_tables.shape[1], 7, nent=lay.num_entries, fills=lay.fills,
               bt=lay.block_tables, dirs=lay.dirs)
    check_structure(gp, lay.lens, 2, 16, nent=lay.num_entries)
    check_entries(gp, lay.lens, 2, 16, lay.block_tables, lay.dirs, nent=lay.num_entries, fills=lay.fills)
    # empty requests, one very long request, single warp ranges of one block
    lens = rng.integers(0, 300, size=40).astype(np.int32)
    lens[rng.integers(0, 40, size=6)] = 0
    lens[3] = 8192
    bt, dirs = synth_map(lens, 512)
    for sms in (1, 2, 148):
        p = _plan(lens, 3, 1, 16, 512, sms)
        check_structure(p, lens, 3, 16)
        check_entries(p, lens, 3, 16, bt, dirs)
    check_structure(_plan(np.zeros(5, np.int32), 2, 1, 16, 4, 148), np.zeros(5, np.int32), 2, 16)


@pytest.mark.parametrize("sms,H,g,bs,general", [(3, 2, 4, 16, False), (1, 1, 8, 16, False),
                                                (5, 3, 1, 32, False), (2, 2, 2, 16, True), (148, 1, 8, 16, False)])
def test_plan_execution_model_matches_dense_attention(sms, H, g, bs, general):
    rng = np.random.default_rng(sms * 7 + H)
    B, d = 12, 8
    lens = rng.integers(1, 200, size=B).astype(np.int32)
    lens[2] = 0
    lens[5] = 1000
    nent = fills = None
    if general:   # random partly filled entries (f3): fills in [1, bs], summing to L
        fl = []
        for L in lens:
            f = []
            while sum(f) < L:
                f.append(int(min(rng.integers(1, bs + 1), L - sum(f))))
            fl.append(f)
        M = max(len(f) for f in fl)
        fills = np.zeros((B, M), np.uint8)
        for r, f in enumerate(fl):
            fills[r, :len(f)] = f
        nent = np.array([len(f) for f in fl], np.int32)
    K = [rng.standard_normal((int(L), H, d)) for L in lens]
    V = [rng.standard_normal((int(L), H, d)) for L in lens]
    q = rng.standard_normal((B, H * g, d))
    bt_stride = int(max(entries(lens, bs, nent).max(), 1))
    plan = _plan(lens, H, g, bs, bt_stride, sms, nent=nent, fills=fills, d=64)
    check_structure(plan, lens, H, bs, nent)
    sim = simulate(plan, lens, H, g, bs, q, K, V, nent, fills)
    ref = dense_attention(lens, H, g, q, K, V)
    assert not np.isnan(sim).any()
    assert np.abs(sim - ref).max() <= 1e-12


def test_plan_rejects_bad_input():
    with pytest.raises(bkv.BkvError):
        _plan(np.array([10, -1], np.int32), 1, 1, 16, 4, 148)
    bt, dirs = synth_map([40], 4)
    with pytest.raises(bkv.BkvError, match="block id"):
        _plan(np.array([40], np.int32), 1, 1, 16, 4, 148, bt=bt - 10 ** 6, dirs=dirs)
    with pytest.raises(bkv.BkvError, match="direction"):
        _plan(np.array([40], np.int32), 1, 1, 16, 4, 148, bt=bt, dirs=dirs + 2)
    with pytest.raises(bkv.BkvError, match="fills"):   # fills summing to 33, not 40
        _plan(np.array([40], np.int32), 1, 1, 16, 4, 148, bt=bt, dirs=dirs,
              fills=np.array([[16, 16, 1, 0]], np.uint8), nent=np.array([3], np.int32))
    with pytest.raises(bkv.BkvError):      # needs 3 entries > bt_stride 2
        _plan(np.array([40], np.int32), 1, 1, 16, 2, 148)
    with pytest.raises(bkv.BkvError):      # group 32 > 16
        _plan(np.array([40], np.int32), 1, 32, 16, 4, 148)


def test_plan_layout_is_fixed_by_geometry():
    """Graph safety: offsets and size depend on (num_seqs, kv heads, SM count) only, so a
    captured graph replays any later plan of the same geometry from the same buffer."""
    rng = np.random.default_rng(7)
    plans = [_plan(rng.integers(0, 3000, 64).astype(np.int32), 2, 8, 16, 256, 148) for _ in range(4)]
    plans.append(_plan(np.zeros(64, np.int32), 2, 8, 16, 256, 148))
    plans.append(_plan(np.full(64, 4096, np.int32), 2, 8, 16, 256, 148))
    hs = [decode(p)[0] for p in plans]
    keys = ("off_wseg", "off_segs", "off_ctask", "off_tasks", "off_zero", "off_xrows", "off_ent")
    assert all(len(p) == len(plans[0]) for p in plans)
    assert all({k: h[k] for k in keys} == {k: hs[0][k] for k in keys} for h in hs)
    assert all(h["n_xrows"] <= h["grid"] for h in hs)
