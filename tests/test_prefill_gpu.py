"""GPU parity of mixed prefill + decode attention through the C ABI.

bkv_paged_prefill_attention against oracle.prefill_attention on the same
seeded inputs (synth: lengths, layouts, K/V, prefill-query stream), dense and
general maps, MHA and GQA, d 64/128, bs 16/32, mixed decode (n = 1) and
prefill rows, poisoned peer slots.  Tolerance: north_star's max-abs 2e-2 /
mean-abs 2e-3 (bf16 inputs, fp32 accumulation).
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2504_09590_b200 as bkv
from synth import make_case
from synth.values import BF16_NAN
from synth.workload import Shape
from tests._cases import dense_case, default_scale
from tests.test_gpu_parity import DEV, check_close, gpu_map, gpu_pool_from_dense, t_u16, u16
from tests.test_general_map_gpu import gmap, gpu_general_pool
from tests.test_prefill_oracle import make_q, pools, query_counts, run_oracle

pytestmark = pytest.mark.gpu


def _run(case, general, n, fill=BF16_NAN, qs=1):
    sh, lay = case.shape, case.layout
    ks, vs, K, V = pools(case, general)
    q, cu = make_q(case, n, sh.num_q_heads, scale_log2=qs)
    ref = run_oracle(case, K, V, cu, q, general)
    if general:
        pool, _ = gpu_general_pool(case, ks, vs, sh.num_kv_heads, fill=fill)
        bt, dirs, lens, fills, nent = gmap(lay)
        kw = dict(fills=fills, num_entries=nent)
    else:
        pool, _ = gpu_pool_from_dense(case, ks, vs, sh.num_kv_heads, fill=fill)
        bt, dirs, lens = gpu_map(lay)
        kw = {}
    o = bkv.paged_prefill_attention(pool, bt, dirs, lens, torch.from_numpy(cu).to(DEV), t_u16(q),
                                    softmax_scale=default_scale(sh.head_dim), **kw)
    torch.cuda.synchronize()
    return o, ref


@pytest.mark.parametrize("cfg,seed,general,full", [("tiny", 0, False, False), ("tiny", 1, True, False),
                                                   ("tiny_gqa", 2, False, False), ("tiny_gqa", 3, True, False),
                                                   ("tiny", 4, False, True), ("tiny_gqa", 5, True, True)])
def test_prefill_parity_small(cfg, seed, general, full):
    case = make_case(cfg, seed, general=general)
    n = query_counts(case.layout.lens, np.random.default_rng(seed), full=full)
    o, ref = _run(case, general, n)
    check_close(o, ref, cfg)


@pytest.mark.parametrize("hq,hkv,d,bs,general", [(8, 1, 128, 16, False), (6, 2, 64, 32, True),
                                                 (5, 5, 128, 32, False), (16, 2, 128, 16, True),
                                                 (12, 4, 64, 16, False)])
def test_prefill_parity_geometries(hq, hkv, d, bs, general):
    sh = Shape("pg", hq, hkv, d, bs, 10, 0.5, "uniform", 900, 1, 1, uniform_max=900)
    case = make_case(sh, hq * 3 + bs, general=general, share_prob=0.9)
    n = query_counts(case.layout.lens, np.random.default_rng(hq), decode_frac=0.3)
    o, ref = _run(case, general, n, qs=2)
    check_close(o, ref, str((hq, hkv, d, bs, general)))


def test_prefill_single_queries_match_decode_kernel():
    """n = 1 everywhere: the prefill kernel is a decode kernel (tolerance, and vs the oracle)."""
    case = make_case("tiny_gqa", 7)
    sh, lay = case.shape, case.layout
    n = np.ones(lay.batch, np.int32)
    o, ref = _run(case, False, n, qs=0)
    check_close(o, ref, "n=1")
    ks, vs, q = dense_case(case)
    pool, _ = gpu_pool_from_dense(case, ks, vs, sh.num_kv_heads)
    bt, dirs, lens = gpu_map(lay)
    od = bkv.paged_decode_attention(pool, bt, dirs, lens, t_u16(q))
    cu = torch.arange(lay.batch + 1, dtype=torch.int32, device=DEV)
    op = bkv.paged_prefill_attention(pool, bt, dirs, lens, cu, t_u16(q))
    torch.cuda.synchronize()
    assert (op.float() - od.float()).abs().max().item() <= 2e-2


def test_prefill_poison_and_zero_query_requests():
    """NaN vs zero in non-owned slots: bitwise equal output; n = 0 rows untouched."""
    case = make_case("tiny_gqa", 8, general=True, share_prob=1.0)
    lay = case.layout
    n = query_counts(lay.lens, np.random.default_rng(8))
    n[::3] = 0
    o1, ref = _run(case, True, n, fill=BF16_NAN)
    o2, _ = _run(case, True, n, fill=0)
    check_close(o1, ref, "poison")
    assert torch.equal(o1.view(torch.int16), o2.view(torch.int16))


def test_prefill_long_context_llama_shard():
    """Llama-70B TP8 shard (1 kv head, 8 q heads): long causal prefill chunks over a
    ShareGPT-like context with shared tails (several 128-row tiles per request)."""
    case = make_case("llama70b", 9)
    sh, lay = case.shape, case.layout
    keep = 24                                   # bounded oracle cost: first 24 requests
    from synth.workload import build_layout, Case
    lay2 = build_layout(lay.lens[:keep], lay.is_be[:keep], 16, np.random.default_rng(3), spare_blocks=2)
    sh1 = Shape("l8", 8, 1, 128, 16, keep, 0.5, "sharegpt", 4096, 1, 8)
    case2 = Case(sh1, lay2, 9)
    n = np.minimum(lay2.lens, np.random.default_rng(4).integers(1, 300, keep)).astype(np.int32)
    o, ref = _run(case2, False, n, qs=0)
    check_close(o, ref, "llama shard")


@pytest.mark.parametrize("cfg,general,pdl", [("tiny_gqa", False, False), ("tiny", True, False),
                                             ("tiny_gqa", False, True), ("tiny", True, True)])
def test_mixed_dispatch_matches_oracle(cfg, general, pdl):
    """bkv_paged_mixed_attention: prefill requests first, then one-row decodes.
    pdl=True: the decode part runs alongside the prefill kernel's tail (no grid wait)."""
    case = make_case(cfg, 12, general=general)
    sh, lay = case.shape, case.layout
    B = lay.batch
    P = B // 2
    n = np.ones(B, np.int32)
    n[:P] = np.minimum(lay.lens[:P], 1 + np.arange(P) * 37)
    ks, vs, K, V = pools(case, general)
    q, cu = make_q(case, n, sh.num_q_heads, scale_log2=1)
    ref = run_oracle(case, K, V, cu, q, general)
    if general:
        pool, _ = gpu_general_pool(case, ks, vs, sh.num_kv_heads)
        bt, dirs, lens, fills, nent = gmap(lay)
        kw = dict(fills=fills, num_entries=nent)
    else:
        pool, _ = gpu_pool_from_dense(case, ks, vs, sh.num_kv_heads)
        bt, dirs, lens = gpu_map(lay)
        kw = {}
    o = bkv.paged_mixed_attention(pool, bt, dirs, lens, torch.from_numpy(cu).to(DEV), t_u16(q), P, int(cu[P]),
                                  softmax_scale=default_scale(sh.head_dim), pdl=pdl, **kw)
    torch.cuda.synchronize()
    check_close(o, ref, cfg)
    if pdl:   # replayed in a CUDA graph, back to back: bit-identical to the eager call
        cu_d, q_d = torch.from_numpy(cu).to(DEV), t_u16(q)
        ws = bkv.workspace(max(1, B - P), sh.num_q_heads, sh.num_kv_heads, sh.head_dim, torch.device(DEV))
        og = torch.empty_like(o)
        mq = int((cu[1:] - cu[:-1]).max())
        fn = lambda: bkv.paged_mixed_attention(pool, bt, dirs, lens, cu_d, q_d, P, int(cu[P]), out=og, ws=ws,
                                               max_q_len=mq, max_seq_len=int(lay.lens.max()),
                                               softmax_scale=default_scale(sh.head_dim), pdl=True, **kw)
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(3):
                fn()
        og.zero_()
        g.replay()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(og, o), "graph replay of the PDL mixed dispatch differs from the eager call"


@pytest.mark.parametrize("cfg,general,full", [("tiny_gqa", False, False), ("tiny_gqa", True, True)])
def test_prefill_mma_sync_kernel_parity_d128(cfg, general, full, monkeypatch):
    """The mma.sync prefill kernel at head_dim 128 (BKV_PREFILL_MMA_SYNC=1; the default there
    is the tcgen05 kernel, which every other d128 test here exercises)."""
    monkeypatch.setenv("BKV_PREFILL_MMA_SYNC", "1")
    case = make_case(cfg, 21, general=general)
    n = query_counts(case.layout.lens, np.random.default_rng(21), full=full)
    o, ref = _run(case, general, n)
    check_close(o, ref, cfg + " mma.sync d128")


def test_prefill_tcgen05_long_context_and_geometries():
    for hq, hkv, bs, general in ((8, 1, 16, False), (16, 2, 32, True), (5, 5, 16, True)):
        sh = Shape("tc", hq, hkv, 128, bs, 8, 0.5, "uniform", 1500, 1, 1, uniform_max=1500)
        case = make_case(sh, hq + bs, general=general, share_prob=0.9)
        n = query_counts(case.layout.lens, np.random.default_rng(hq), decode_frac=0.3)
        o, ref = _run(case, general, n, qs=2)
        check_close(o, ref, str((hq, hkv, bs, general)))


@pytest.mark.parametrize("cfg,general", [("tiny_gqa", False), ("tiny_gqa", True)])
def test_prefill_tcgen05_single_query_tile_per_cta(cfg, general, monkeypatch):
    """BKV_PREFILL_QT=1: the tcgen05 kernel with one 128-row query tile per CTA (the
    default runs two ping-pong tiles per CTA)."""
    monkeypatch.setenv("BKV_PREFILL_QT", "1")
    case = make_case(cfg, 31, general=general)
    n = query_counts(case.layout.lens, np.random.default_rng(31))
    o, ref = _run(case, general, n)
    check_close(o, ref, cfg + " QT1")


@pytest.mark.parametrize("seed", range(8))
def test_prefill_random_geometry_fuzz(seed, monkeypatch):
    """Seeded random geometries (group size, head_dim 64/128 -> mma.sync / tcgen05 kernels,
    block size, batch, dense or general map, whole-prompt / suffix / decode rows), and on
    odd seeds the tcgen05 kernel with one query tile per CTA, against the oracle."""
    if seed % 2:
        monkeypatch.setenv("BKV_PREFILL_QT", "1")
    rng = np.random.default_rng(3000 + seed)
    hkv = int(rng.choice([1, 2, 4]))
    g = int(rng.choice([1, 2, 4, 8, 16]))
    d = int(rng.choice([64, 128]))
    bs = int(rng.choice([16, 32]))
    B = int(rng.integers(1, 24))
    general = bool(rng.random() < 0.5)
    sh = Shape(f"pfuzz{seed}", hkv * g, hkv, d, bs, B, 0.5, "uniform", 900, 1, 1, uniform_max=900)
    case = make_case(sh, seed, general=general)
    n = query_counts(case.layout.lens, rng, full=bool(rng.random() < 0.3))
    o, ref = _run(case, general, n, qs=int(rng.integers(0, 3)))
    check_close(o, ref, f"pfuzz{seed} g{g} hkv{hkv} d{d} bs{bs} B{B} general{general}")


@pytest.mark.parametrize("q_ldg,o_stg", [(1, 0), (0, 1), (1, 1)])
def test_prefill_tcgen05_q_and_output_fallbacks(q_ldg, o_stg, monkeypatch):
    """The tcgen05 kernel's load/store fallbacks forced at g = 8: Q staged by the softmax warps
    (BKV_PREFILL_Q_LDG=1, the path of group sizes not dividing 128) and output rows stored
    directly (BKV_PREFILL_O_STG=1, the path of group sizes not dividing 32)."""
    monkeypatch.setenv("BKV_PREFILL_Q_LDG", str(q_ldg))
    monkeypatch.setenv("BKV_PREFILL_O_STG", str(o_stg))
    for general in (False, True):
        case = make_case("tiny_gqa", 41 + q_ldg + 2 * o_stg, general=general)
        n = query_counts(case.layout.lens, np.random.default_rng(41), full=general)
        o, ref = _run(case, general, n)
        check_close(o, ref, f"tiny_gqa q_ldg{q_ldg} o_stg{o_stg} general{general}")


@pytest.mark.parametrize("hq,hkv", [(6, 2), (10, 2), (12, 2)])
def test_prefill_tcgen05_group_sizes_not_dividing_tiles(hq, hkv):
    """Group sizes 3, 5, 6: a 128-row query tile (and a warp's 32 rows) starts mid-token, so
    the kernel takes its load-staged Q and direct-store output paths (no TMA row boxes)."""
    sh = Shape(f"g{hq // hkv}", hq, hkv, 128, 16, 6, 0.5, "uniform", 700, 1, 1, uniform_max=700)
    case = make_case(sh, hq, general=True)
    n = query_counts(case.layout.lens, np.random.default_rng(hq), decode_frac=0.3)
    o, ref = _run(case, True, n)
    check_close(o, ref, f"g{hq // hkv}")


@pytest.mark.parametrize("hkv,dispatch", [(1, False), (1, True), (8, True)])
def test_prefill_bench_workload_every_element(hkv, dispatch):
    """bench_prefill.py's mixed batch at the Llama-70B TP8 (1 kv head, 8 q heads) and TP1
    (8 kv heads, 64 q heads: the headline prefill measurement) shard shapes:
    the llama70b seed-0 layout (batch 256), 16 BE requests prefilling their whole prompt
    (rng seed 1, as the bench picks them) and every other request decoding one token; every
    output element vs the oracle.  dispatch: the bench's default path -- prefill requests
    moved first, bkv_paged_mixed_attention (prefill kernel + split-K decode kernel) --
    else one bkv_paged_prefill_attention over the batch in layout order."""
    from dataclasses import replace
    from synth.workload import Case
    base = make_case("llama70b", 0)
    lay = base.layout
    rng = np.random.default_rng(1)
    be = np.flatnonzero(lay.is_be)
    pre = rng.choice(be, size=min(16, be.size), replace=False)
    n = np.ones(lay.batch, np.int32)
    n[pre] = lay.lens[pre]
    if dispatch:
        perm = np.concatenate([pre, np.setdiff1d(np.arange(lay.batch), pre)])
        lay = replace(lay, lens=lay.lens[perm], is_be=lay.is_be[perm], block_tables=lay.block_tables[perm],
                      dirs=lay.dirs[perm])
        n = n[perm]
    sh = Shape("l70bench", 8 * hkv, hkv, 128, 16, lay.batch, 0.5, "sharegpt", 4096, 1, 8 // hkv)
    case = Case(sh, lay, 0)
    ks, vs, K, V = pools(case, False)
    q, cu = make_q(case, n, 8 * hkv)
    ref = run_oracle(case, K, V, cu, q, False)
    pool, _ = gpu_pool_from_dense(case, ks, vs, hkv)
    bt, dirs, lens = gpu_map(lay)
    cu_d = torch.from_numpy(cu).to(DEV)
    if dispatch:
        P = len(pre)
        o = bkv.paged_mixed_attention(pool, bt, dirs, lens, cu_d, t_u16(q), P, int(cu[P]),
                                      max_q_len=int(n[:P].max()), max_seq_len=int(lay.lens.max()),
                                      softmax_scale=default_scale(128), pdl=True)
    else:
        o = bkv.paged_prefill_attention(pool, bt, dirs, lens, cu_d, t_u16(q), max_q_len=int(n.max()),
                                        softmax_scale=default_scale(128))
    torch.cuda.synchronize()
    check_close(o, ref, f"bench workload hkv={hkv} dispatch={dispatch}")


@pytest.mark.parametrize("batch", [511, 512, 513, 700])
def test_prefill_many_requests_zero_rows(batch):
    """Batches around the kernel's live-request compaction limit (512 requests): up to it the
    work items enumerate only requests with rows, beyond it every request; a third of the
    requests have no rows, the rest decode or prefill a suffix."""
    sh = Shape(f"many{batch}", 8, 1, 128, 16, batch, 0.5, "uniform", 160, 1, 8, uniform_max=160)
    case = make_case(sh, batch, general=bool(batch % 2))
    rng = np.random.default_rng(batch)
    n = query_counts(case.layout.lens, rng, decode_frac=0.4)
    n[rng.random(batch) < 0.33] = 0
    o, ref = _run(case, bool(batch % 2), n)
    check_close(o, ref, f"batch {batch}")
