"""GPU parity of the planned decode (bkv_decode_plan + bkv_decode_planned, one launch per
layer) against the CPU oracle, through the C ABI.

Attention within max-abs 2e-2 / mean-abs 2e-3 of the fp64 oracle over EVERY output
element (BASELINE.json north_star); the fused append and the pool bit-exact; repeated
calls bitwise identical (the merge order is fixed by the plan, the cross-CTA counters
clean themselves up).
"""
import math

import numpy as np
import pytest
import torch

import oracle
import paper_2504_09590_b200 as bkv
from synth import make_case, build_layout
from synth.values import BF16_NAN
from synth.workload import Shape, Case, sweep_shape
from tests._cases import dense_case, oracle_pool, ragged, default_scale
from tests._full import run_full
from tests.test_gpu_parity import (t_u16, u16, gpu_map, gpu_pool_from_dense, check_close, ATT_CASES, DEV,
                                   MAX_ABS)

pytestmark = pytest.mark.gpu


def _planned_case(case, per_request=False, fill=BF16_NAN, out=None, general=False, peers=0, repeat=1):
    sh, lay = case.shape, case.layout
    ks, vs, q = dense_case(case)
    gmn = dict(fills=lay.fills, num_entries=lay.num_entries) if general else {}
    K, V = oracle.new_pool(lay.num_blocks, sh.num_kv_heads, sh.block_size, sh.head_dim, BF16_NAN)
    kn, vn, cu = ragged(ks, vs, lay.lens, np.zeros(lay.batch, np.int32))
    dirs_np = lay.dirs_per_request if per_request else lay.dirs
    oracle.append(K, V, lay.block_tables, dirs_np, np.zeros(lay.batch, np.int32), cu, kn, vn, **gmn)
    ref = oracle.attention(K, V, lay.block_tables, dirs_np, lay.lens, q, default_scale(sh.head_dim), **gmn)
    pool = bkv.KVPool(t_u16(K if fill == BF16_NAN else np.where(K == BF16_NAN, np.uint16(fill), K)),
                      t_u16(V if fill == BF16_NAN else np.where(V == BF16_NAN, np.uint16(fill), V)))
    bt, dirs, lens = gpu_map(lay, per_request)
    gm = {k: torch.from_numpy(v).to(DEV) for k, v in gmn.items()}
    plan = bkv.decode_plan(lay.lens, lay.block_tables, dirs_np, pool, sh.num_q_heads,
                           fills_host=lay.fills if general else None,
                           num_entries_host=lay.num_entries if general else None)
    peer_bufs = [torch.full((lay.batch, sh.num_q_heads, sh.head_dim), float("nan"), dtype=torch.bfloat16,
                            device=DEV) for _ in range(peers)]
    outs = [bkv.decode_planned(pool, bt, dirs, lens, plan, t_u16(q), out=out, peer_outs=peer_bufs, **gm).clone()
            for _ in range(repeat)]
    torch.cuda.synchronize()
    for o in outs[1:]:
        assert torch.equal(o.view(torch.int16), outs[0].view(torch.int16))
    for pb in peer_bufs:
        assert torch.equal(pb.view(torch.int16), outs[0].contiguous().view(torch.int16))
    return outs[0], ref


@pytest.mark.parametrize("cfg,seed,qs", ATT_CASES)
def test_planned_parity_small(cfg, seed, qs):
    o, ref = _planned_case(make_case(cfg, seed, q_scale_log2=qs), repeat=3)
    check_close(o, ref, cfg)


@pytest.mark.parametrize("hq,hkv,d,bs", [(16, 1, 128, 16), (12, 1, 64, 32), (6, 2, 64, 16),
                                         (3, 3, 64, 32), (5, 5, 128, 32), (32, 2, 128, 16), (8, 8, 128, 16)])
def test_planned_parity_geometries(hq, hkv, d, bs):
    sh = Shape("geo", hq, hkv, d, bs, 20, 0.5, "uniform", 700, 1, 1, uniform_max=700)
    o, ref = _planned_case(make_case(sh, hq * 7 + bs, q_scale_log2=2))
    check_close(o, ref, str((hq, hkv, d, bs)))


@pytest.mark.parametrize("direction", [0, 1])
def test_planned_edge_lengths_and_empty(direction):
    lens = [1, 0, 2, 15, 16, 17, 31, 32, 33, 0, 47, 48, 63, 64, 65, 255, 256, 257, 1000, 2049, 0]
    for hq, hkv, d, bs in ((8, 2, 128, 16), (4, 4, 64, 32), (16, 1, 128, 32)):
        sh = Shape("edge", hq, hkv, d, bs, len(lens), 0.5, "uniform", 4096, 1, 1)
        case = make_case(sh, 4 + direction, lens=lens, is_be=[bool(direction)] * len(lens))
        o, ref = _planned_case(case)
        check_close(o, ref, f"{(hq, hkv, d, bs)} dir{direction}")
        assert (u16(o)[[i for i, L in enumerate(lens) if L == 0]] == 0).all(), "empty context -> zeros (Q8)"


@pytest.mark.parametrize("L,hq,hkv,bs", [(8192, 8, 1, 16), (30000, 8, 1, 32), (4096, 4, 4, 16)])
def test_planned_one_long_request_spans_every_cta(L, hq, hkv, bs):
    """One request: its row(s) are cut across every warp of the grid (P = 1-2 blocks per
    warp), so the cross-CTA merge combines up to 148 CTA pieces in batches of 8."""
    sh = Shape("long", hq, hkv, 128, bs, 1, 0.5, "uniform", L, 1, 1)
    case = make_case(sh, 9, lens=[L], is_be=[True])
    o, ref = _planned_case(case, repeat=2)
    check_close(o, ref, f"long L={L} g={hq // hkv} bs={bs}")


def test_planned_single_token_is_exact_v0():
    for hq, hkv, d in ((4, 4, 64), (8, 1, 128), (16, 2, 128)):
        sh = Shape("one", hq, hkv, d, 16, 6, 0.5, "uniform", 16, 1, 1)
        case = make_case(sh, 1, lens=[1] * 6)
        o, _ = _planned_case(case)
        _, vs, _ = dense_case(case)
        exp = np.stack([np.stack([vs[r][0, h // (hq // hkv)] for h in range(hq)]) for r in range(6)])
        assert np.array_equal(u16(o), exp)


def test_planned_poison_head_major_per_request_peers():
    case = make_case("tiny_gqa", 12)
    sh, lay = case.shape, case.layout
    o1, ref = _planned_case(case, fill=BF16_NAN)
    o2, _ = _planned_case(case, fill=0)
    check_close(o1, ref, "poison")
    assert torch.equal(o1.view(torch.int16), o2.view(torch.int16)), "P5(vi): non-owned slots never matter"
    out = torch.empty((sh.num_q_heads, lay.batch, sh.head_dim), dtype=torch.bfloat16, device=DEV).permute(1, 0, 2)
    o3, _ = _planned_case(case, per_request=True, out=out)
    check_close(o3, ref, "head-major, per-request flags")
    o4, _ = _planned_case(case, peers=3)   # fused reassembly: peers get bitwise copies
    assert torch.equal(o4.view(torch.int16), o1.view(torch.int16))


@pytest.mark.parametrize("seed", range(3))
def test_planned_general_map(seed):
    case = make_case("tiny_gqa", seed, general=True, share_prob=0.9)
    o, ref = _planned_case(case, general=True)
    check_close(o, ref, f"general{seed}")


def test_planned_fused_step_bitwise_pool():
    """bkv_decode_planned with k_new/v_new == bkv_decode_step: the pool bit-exact vs the
    oracle append, outputs within tolerance of the oracle."""
    sh = Shape("ps", 16, 2, 128, 16, 24, 0.5, "uniform", 600, 1, 1, uniform_max=600)
    case = make_case(sh, 31)
    lay = case.layout
    ks, vs, q = dense_case(case)
    B = lay.batch
    before = (lay.lens - 1).astype(np.int32)
    Kp, Vp = oracle.new_pool(lay.num_blocks, 2, 16, 128, BF16_NAN)
    kn, vn, cu = ragged(ks, vs, before, np.zeros(B, np.int32))
    oracle.append(Kp, Vp, lay.block_tables, lay.dirs, np.zeros(B, np.int32), cu, kn, vn)
    pool = bkv.KVPool(t_u16(Kp), t_u16(Vp))
    kd, vd, cud = ragged(ks, vs, lay.lens, before)
    oracle.append(Kp, Vp, lay.block_tables, lay.dirs, before, cud, kd, vd)
    ref = oracle.attention(Kp, Vp, lay.block_tables, lay.dirs, lay.lens, q, default_scale(128))
    bt, dirs, lens = gpu_map(lay)
    plan = bkv.decode_plan(lay.lens, lay.block_tables, lay.dirs, pool, 16)
    o = bkv.decode_planned(pool, bt, dirs, lens, plan, t_u16(q), k_new=t_u16(kd), v_new=t_u16(vd), pdl=True)
    torch.cuda.synchronize()
    assert np.array_equal(u16(pool.k), Kp) and np.array_equal(u16(pool.v), Vp)
    check_close(o, ref, "planned step")


# ----------------------------------------------- full size: every element, every pool byte
@pytest.mark.parametrize("cfg,tp,rank", [("opt13b", 1, 0), ("llama70b", 1, 0), ("llama70b", 8, 0),
                                         ("llama70b", 8, 7), ("llama70b", 4, 1), ("llama70b", 2, 0),
                                         ("opt13b", 2, 1), ("opt13b", 8, 3), ("opt30b", 4, 2)])
def test_planned_full_size_every_element(cfg, tp, rank):
    """The bench's launch configuration (fused step, PDL) at the BASELINE batch, seed 0 (the
    bench's seed): every output element vs the oracle, every pool byte after the append."""
    _, _, per_req = run_full(cfg, tp, rank, seed=0, mode="step", pdl=True, planned=True, repeat=2)
    assert per_req.max() <= MAX_ABS


def test_planned_full_size_general_map_and_attn_mode():
    run_full("llama70b", 8, 2, seed=3, mode="step", planned=True, general=True)
    run_full("opt13b", 4, 0, seed=4, mode="attn", planned=True)


@pytest.mark.parametrize("L0,bs,rt,tp", [(8192, 32, 0.25, 8), (8192, 16, 1.0, 8), (512, 16, 0.0, 8),
                                         (2048, 32, 0.75, 4), (4096, 16, 0.5, 2)])
def test_planned_sweep_configs(L0, bs, rt, tp):
    """BASELINE configs[4] (Llama-2-70B shape, 512-8K contexts, bs 16/32, RT:BE mix) at TP shards."""
    run_full(sweep_shape(L0, bs, rt), tp, 1, seed=2, mode="step", planned=True, check_pool=False)


def test_planned_rejects_mismatched_plan():
    case = make_case("tiny_gqa", 3)
    sh, lay = case.shape, case.layout
    pool = bkv.KVPool.empty(lay.num_blocks, sh.num_kv_heads, sh.block_size, sh.head_dim, DEV)
    bt, dirs, lens = gpu_map(lay)
    q = torch.zeros((lay.batch, sh.num_q_heads, sh.head_dim), dtype=torch.bfloat16, device=DEV)
    plan = bkv.decode_plan(lay.lens, lay.block_tables, lay.dirs, (sh.num_kv_heads * 2, sh.head_dim, sh.block_size),
                           sh.num_q_heads * 2)
    with pytest.raises(bkv.BkvError, match="does not match"):
        bkv.decode_planned(pool, bt, dirs, lens, plan, q)
    other = bkv.decode_plan_host(lay.lens, lay.block_tables, lay.dirs, sh.num_kv_heads, sh.num_q_heads,
                                 sh.head_dim, sh.block_size, num_sms=7)
    bad = bkv.DecodePlan(other, plan.dev, plan.nbytes)
    with pytest.raises(bkv.BkvError, match="warps"):
        bkv.decode_planned(pool, bt, dirs, lens, bad, q)


def test_planned_graph_replays_a_new_plan():
    """A CUDA graph captured with step A's plan replays step B (new lengths, same batch and
    geometry) once B's plan and lengths are copied into the same device buffers: equal to an
    eager call with plan B (graph safety of the fixed-capacity plan layout)."""
    sh = Shape("gr", 16, 2, 128, 16, 40, 0.5, "uniform", 900, 1, 1, uniform_max=900)
    case_b = make_case(sh, 77)
    lay = case_b.layout
    ks, vs, q = dense_case(case_b)
    K, V, _ = oracle_pool(case_b, ks, vs, 2)
    ref = oracle.attention(K, V, lay.block_tables, lay.dirs, lay.lens, q, default_scale(128))
    pool = bkv.KVPool(t_u16(K), t_u16(V))
    bt, dirs, lens = gpu_map(lay)
    lens_a = np.maximum(1, lay.lens // 3).astype(np.int32)          # step A: shorter contexts
    plan = bkv.decode_plan(lens_a, lay.block_tables, lay.dirs, pool, 16)
    lens.copy_(torch.from_numpy(lens_a))
    qd = t_u16(q)
    out = torch.empty_like(qd)
    ws = bkv.workspace(lay.batch, 16, 2, 128)
    bkv.decode_planned(pool, bt, dirs, lens, plan, qd, out=out, ws=ws, pdl=True)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        bkv.decode_planned(pool, bt, dirs, lens, plan, qd, out=out, ws=ws, pdl=True)
    plan_b = bkv.decode_plan_host(lay.lens, lay.block_tables, lay.dirs, 2, 16, 128, 16)
    assert plan_b.nbytes == plan.host.nbytes
    plan.upload(plan_b)
    lens.copy_(torch.from_numpy(lay.lens.astype(np.int32)))
    g.replay()
    torch.cuda.synchronize()
    check_close(out, ref, "graph replay with plan B")
    eager = bkv.decode_planned(pool, bt, dirs, lens, plan, qd)
    torch.cuda.synchronize()
    assert torch.equal(eager.view(torch.int16), out.view(torch.int16))


def test_planned_dynamic_dispatch(monkeypatch):
    """Plans with long warp ranges (>= BKV_PLANNED_DYNAMIC_P blocks per warp; 128 by default,
    e.g. OPT-30B on one GPU) run the dynamically scheduled kernel pair: forced here for a
    full-size Llama-70B TP8 shard and the small cases -- every element vs the oracle."""
    monkeypatch.setenv("BKV_PLANNED_DYNAMIC_P", "1")
    run_full("llama70b", 8, 4, seed=6, mode="step", planned=True, repeat=2)
    for cfg_s, seed, qs in ATT_CASES:
        o, ref = _planned_case(make_case(cfg_s, seed, q_scale_log2=qs))
        check_close(o, ref, cfg_s)
