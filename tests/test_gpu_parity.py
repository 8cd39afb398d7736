"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Both sides consume the same seeded synthetic inputs (synth/).  Append and the
slot map must match bit for bit; attention within max-abs 2e-2 / mean-abs 2e-3
of the fp64 oracle (BASELINE.json north_star).
"""
import math
import os

import numpy as np
import pytest
import torch

import oracle
import paper_2504_09590_b200 as bkv
from synth import CONFIGS, make_case, build_layout, dense_kv_torch, q_torch
from synth.values import BF16_NAN
from synth.workload import Shape, shard_heads
from tests._cases import dense_case, oracle_pool, ragged, default_scale
from tests._full import run_full

pytestmark = pytest.mark.gpu

MAX_ABS, MEAN_ABS = 2e-2, 2e-3
DEV = "cuda"


def t_u16(a):
    """numpy uint16 bf16 bits -> torch bf16 on the GPU."""
    return torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).to(DEV).view(torch.bfloat16)


def u16(t):
    return t.detach().view(torch.int16).cpu().numpy().view(np.uint16)


def gpu_map(lay, per_request=False):
    bt = torch.from_numpy(lay.block_tables).to(DEV)
    dirs = torch.from_numpy(lay.dirs_per_request if per_request else lay.dirs).to(DEV)
    return bt, dirs, torch.from_numpy(lay.lens.astype(np.int32)).to(DEV)


def gpu_pool_from_dense(case, ks, vs, n_heads, fill=BF16_NAN, per_request=False):
    sh, lay = case.shape, case.layout
    pool = bkv.KVPool.empty(lay.num_blocks, n_heads, sh.block_size, sh.head_dim, DEV)
    pool.k.view(torch.int16).fill_(np.int16(np.uint16(fill).view(np.int16)))
    pool.v.view(torch.int16).fill_(np.int16(np.uint16(fill).view(np.int16)))
    before = np.zeros(lay.batch, np.int32)
    kn, vn, cu = ragged(ks, vs, lay.lens, before)
    bt, dirs, _ = gpu_map(lay, per_request)
    sm = torch.zeros(kn.shape[0], dtype=torch.int64, device=DEV)
    bkv.kv_append(pool, bt, dirs, torch.from_numpy(before).to(DEV), torch.from_numpy(cu).to(DEV),
                  t_u16(kn), t_u16(vn), slot_mapping=sm)
    return pool, sm


def check_close(out_gpu, ref, tag=""):
    o = out_gpu.float().cpu().numpy().astype(np.float64)
    assert np.isfinite(o).all(), tag
    err = np.abs(o - ref)
    assert err.max() <= MAX_ABS and err.mean() <= MEAN_ABS, (tag, err.max(), err.mean())
    return err


# ------------------------------------------------------------------ append
@pytest.mark.parametrize("cfg,seed,per_request", [("tiny", 0, False), ("tiny", 1, True),
                                                  ("tiny_gqa", 2, False), ("llama70b", 3, False)])
def test_kv_append_bitwise(cfg, seed, per_request):
    case = make_case(cfg, seed)
    sh, lay = case.shape, case.layout
    heads = list(range(sh.num_kv_heads)) if cfg != "llama70b" else [5]   # TP8 shard of rank 5
    ks, vs, _ = dense_case(case, kv_heads=heads, q_heads=[0])
    Ko, Vo, smo = oracle_pool(case, ks, vs, len(heads), per_request_dirs=per_request)
    pool, sm = gpu_pool_from_dense(case, ks, vs, len(heads), per_request=per_request)
    torch.cuda.synchronize()
    assert np.array_equal(u16(pool.k), Ko) and np.array_equal(u16(pool.v), Vo)
    assert np.array_equal(sm.cpu().numpy(), smo)


def test_kv_append_decode_step_and_bs32():
    """One decode step on top of a prefilled pool, bs = 32, shared RT/BE tails."""
    sh = Shape("t32", 4, 2, 128, 32, 24, 0.5, "uniform", 600, 1, 1, uniform_max=600)
    case = make_case(sh, 8)
    lay = case.layout
    ks, vs, _ = dense_case(case)
    B = lay.batch
    before = (lay.lens - 1).astype(np.int32)
    # prefill tokens [0, L-1) on both sides, then append token L-1 as a decode step
    Ko, Vo = oracle.new_pool(lay.num_blocks, 2, 32, 128, BF16_NAN)
    kn, vn, cu = ragged(ks, vs, before, np.zeros(B, np.int32))
    oracle.append(Ko, Vo, lay.block_tables, lay.dirs, np.zeros(B, np.int32), cu, kn, vn)
    pool = bkv.KVPool(t_u16(Ko.copy()), t_u16(Vo.copy()))
    kd, vd, cud = ragged(ks, vs, lay.lens, before)
    smo = oracle.append(Ko, Vo, lay.block_tables, lay.dirs, before, cud, kd, vd)
    bt, dirs, _ = gpu_map(lay)
    sm = torch.zeros(B, dtype=torch.int64, device=DEV)
    bkv.kv_append(pool, bt, dirs, torch.from_numpy(before).to(DEV), torch.from_numpy(cud).to(DEV),
                  t_u16(kd), t_u16(vd), slot_mapping=sm)
    torch.cuda.synchronize()
    assert np.array_equal(u16(pool.k), Ko) and np.array_equal(u16(pool.v), Vo)
    assert np.array_equal(sm.cpu().numpy(), smo)


# --------------------------------------------------------------- attention
def _run_case(case, per_request=False, fill=BF16_NAN, qscale=None, out=None):
    sh, lay = case.shape, case.layout
    ks, vs, q = dense_case(case)
    K, V, _ = oracle_pool(case, ks, vs, sh.num_kv_heads, per_request_dirs=per_request)
    scale = default_scale(sh.head_dim) if qscale is None else qscale
    ref = oracle.attention(K, V, lay.block_tables, lay.dirs, lay.lens, q, scale)
    pool, _ = gpu_pool_from_dense(case, ks, vs, sh.num_kv_heads, fill=fill, per_request=per_request)
    bt, dirs, lens = gpu_map(lay, per_request)
    o = bkv.paged_decode_attention(pool, bt, dirs, lens, t_u16(q), scale, out=out)
    torch.cuda.synchronize()
    return o, ref, (ks, vs, q, pool)


ATT_CASES = [
    ("tiny", 0, 0), ("tiny", 1, 3), ("tiny_gqa", 2, 0), ("tiny_gqa", 3, 3),
]


@pytest.mark.parametrize("cfg,seed,qs", ATT_CASES)
def test_attention_parity_small(cfg, seed, qs):
    case = make_case(cfg, seed, q_scale_log2=qs)
    o, ref, _ = _run_case(case)
    check_close(o, ref, cfg)


@pytest.mark.parametrize("hq,hkv,d,bs", [(16, 1, 128, 16), (12, 1, 64, 32), (6, 2, 64, 16),
                                         (3, 3, 64, 32), (5, 5, 128, 32), (32, 2, 128, 16)])
def test_attention_parity_geometries(hq, hkv, d, bs):
    """MHA (CUDA cores) and GQA g = 2..16 (MMA) at d 64/128, bs 16/32, ragged lengths."""
    sh = Shape("geo", hq, hkv, d, bs, 20, 0.5, "uniform", 700, 1, 1, uniform_max=700)
    case = make_case(sh, hq * 7 + bs, q_scale_log2=2)
    o, ref, _ = _run_case(case)
    check_close(o, ref, str((hq, hkv, d, bs)))


@pytest.mark.parametrize("direction", [0, 1])
def test_edge_lengths(direction):
    lens = [1, 2, 15, 16, 17, 31, 32, 33, 47, 48, 63, 64, 65, 255, 256, 257, 1000, 2049]
    sh = Shape("edge", 8, 2, 128, 16, len(lens), 0.5, "uniform", 4096, 1, 1)
    case = make_case(sh, 4, lens=lens, is_be=[bool(direction)] * len(lens))
    o, ref, _ = _run_case(case)
    check_close(o, ref, f"dir{direction}")
    sh1 = Shape("edge1", 4, 4, 64, 32, len(lens), 0.5, "uniform", 4096, 1, 1)
    case = make_case(sh1, 5, lens=lens, is_be=[bool(direction)] * len(lens))
    o, ref, _ = _run_case(case)
    check_close(o, ref, f"mha dir{direction}")


def test_streamk_plan_forced_on_small_cases(monkeypatch):
    """Stream-K split plan (equal contiguous block ranges per warp, rows cut across warps,
    pieces merged from per-range slots) forced on for problems the auto rule leaves to the
    bucket plan: MHA and GQA, both directions, empty and ragged contexts, bs 16/32."""
    monkeypatch.setenv("BKV_STREAMK", "2")
    for cfg, seed, qs in ATT_CASES:
        case = make_case(cfg, seed, q_scale_log2=qs)
        o, ref, _ = _run_case(case)
        check_close(o, ref, "stream-K " + cfg)
    lens = [0, 1, 2, 15, 16, 17, 33, 0, 64, 65, 257, 1000, 2049, 0]
    for hq, hkv, d, bs in ((8, 2, 128, 16), (4, 4, 64, 32), (16, 1, 128, 32)):
        sh = Shape("skedge", hq, hkv, d, bs, len(lens), 0.5, "uniform", 4096, 1, 1)
        for direction in (0, 1):
            case = make_case(sh, 6 + direction, lens=lens, is_be=[bool(direction)] * len(lens))
            o, ref, _ = _run_case(case)
            check_close(o, ref, f"stream-K {(hq, hkv, d, bs)} dir{direction}")


@pytest.mark.parametrize("cfg,tp,rank", [("llama70b", 4, 1), ("opt13b", 4, 3), ("llama70b", 2, 0)])
def test_full_size_streamk_auto(cfg, tp, rank):
    """Shards where the auto rule picks the stream-K plan (warp ranges >= 12 blocks), in the
    bench's launch configuration (fused step, PDL), sampled against the oracle."""
    _full_size(cfg, tp, rank, mode="step", pdl=True, seed=4)


def test_single_token_is_exact_v0():
    """Closed form P3(i): L = 1 => out = v_0 bitwise (softmax weight exactly 1)."""
    for hq, hkv, d in ((4, 4, 64), (8, 1, 128), (16, 2, 128)):
        sh = Shape("one", hq, hkv, d, 16, 6, 0.5, "uniform", 16, 1, 1)
        case = make_case(sh, 1, lens=[1] * 6)
        o, ref, (ks, vs, q, _) = _run_case(case)
        exp = np.stack([np.stack([vs[r][0, h // (hq // hkv)] for h in range(hq)]) for r in range(6)])
        assert np.array_equal(u16(o), exp)


def test_per_request_direction_flags_and_head_major_out():
    case = make_case("tiny_gqa", 9)
    sh, lay = case.shape, case.layout
    B = lay.batch
    out = torch.empty((sh.num_q_heads, B, sh.head_dim), dtype=torch.bfloat16, device=DEV).permute(1, 0, 2)
    o, ref, _ = _run_case(case, per_request=True, out=out)
    check_close(o, ref, "head-major")


def test_poisoned_peer_slots_do_not_change_output():
    """P5(vi): NaN in every non-owned slot gives bitwise the same output as zeros."""
    for cfg in ("tiny", "tiny_gqa"):
        case = make_case(cfg, 12)
        o1, ref, _ = _run_case(case, fill=BF16_NAN)
        o2, _, _ = _run_case(case, fill=0)
        check_close(o1, ref, cfg)
        assert torch.equal(o1.view(torch.int16), o2.view(torch.int16))


def test_empty_context_gives_zeros():
    sh = Shape("z", 8, 1, 128, 16, 4, 0.5, "uniform", 64, 1, 1)
    lay = build_layout([0, 5, 0, 40], [False, True, True, False], 16, np.random.default_rng(0), spare_blocks=2)
    from synth.workload import Case
    case = Case(sh, lay, 3)
    o, ref, _ = _run_case(case)
    assert (u16(o)[[0, 2]] == 0).all()
    check_close(o, ref, "zeros")


def test_split_plan_invariance_and_determinism(monkeypatch):
    """P5(v): forcing many tiny splits changes nothing beyond tolerance; repeated
    calls are bitwise identical (fixed merge order, self-resetting workspace)."""
    case = make_case("tiny_gqa", 21)
    o_def, ref, (ks, vs, q, pool) = _run_case(case)
    lay = case.layout
    bt, dirs, lens = gpu_map(lay)
    monkeypatch.setenv("BKV_MIN_SPLIT", "1")
    monkeypatch.setenv("BKV_UNITS_PER_WARP", "64")
    outs = [bkv.paged_decode_attention(pool, bt, dirs, lens, t_u16(q)) for _ in range(3)]
    torch.cuda.synchronize()
    for o in outs:
        check_close(o, ref, "many splits")
        assert torch.equal(o.view(torch.int16), outs[0].view(torch.int16))
    monkeypatch.delenv("BKV_MIN_SPLIT")
    monkeypatch.delenv("BKV_UNITS_PER_WARP")
    o2 = bkv.paged_decode_attention(pool, bt, dirs, lens, t_u16(q))
    torch.cuda.synchronize()
    assert torch.equal(o2.view(torch.int16), o_def.view(torch.int16))


def test_gqa_equals_mha_with_repeated_kv_heads():
    """P5(iii): GQA (MMA path) vs MHA (CUDA-core path) over repeated kv heads."""
    case = make_case("tiny_gqa", 13)
    sh, lay = case.shape, case.layout
    o, ref, (ks, vs, q, pool) = _run_case(case)
    g = sh.group
    pool_r = bkv.KVPool(pool.k.repeat_interleave(g, dim=1).contiguous(), pool.v.repeat_interleave(g, dim=1).contiguous())
    bt, dirs, lens = gpu_map(lay)
    o2 = bkv.paged_decode_attention(pool_r, bt, dirs, lens, t_u16(q))
    torch.cuda.synchronize()
    check_close(o2, ref, "mha-repeat")
    assert (o.float() - o2.float()).abs().max().item() <= 2 * MAX_ABS


# --------------------------------------- full-size configs, every element
def _full_size(cfg, tp=1, rank=0, seed=0, mode="attn", pdl=False, spare_blocks=3, repeat=1, **_):
    """Full BASELINE-size batch on the GPU through the dynamically scheduled kernel pair
    (bkv_paged_decode_attention / bkv_decode_step); every output element -- and for the
    fused step every pool byte -- against the oracle (tests/_full.py)."""
    got, ref, per_req = run_full(cfg, tp, rank, seed=seed, mode=mode, pdl=pdl, planned=False,
                                 spare_blocks=spare_blocks, repeat=repeat)
    return torch.from_numpy(got)


@pytest.mark.parametrize("cfg,tp,rank", [("opt13b", 1, 0), ("opt30b", 4, 2), ("llama70b", 1, 0), ("llama70b", 8, 7)])
def test_full_size_parity(cfg, tp, rank):
    _full_size(cfg, tp, rank)


@pytest.mark.parametrize("cfg,tp", [("opt13b", 1), ("llama70b", 8), ("opt30b", 2)])
def test_full_size_fused_step(cfg, tp):
    """The fused decode step with PDL at the full BASELINE batch, seed 0 (bench.py's seed), twice
    (bitwise repeat); bkv_decode_planned's large-problem path (OPT-30B at one GPU) runs this pair."""
    _full_size(cfg, tp, 0, mode="step", pdl=True, seed=0, repeat=2)


@pytest.mark.parametrize("cfg,tp", [("llama70b", 8), ("opt13b", 4)])
def test_fused_merge_opt_in(cfg, tp, monkeypatch):
    """BKV_FUSED_MERGE=1, the opt-in in-kernel last-arriver merge (group merge for GQA, row
    merge for MHA): sampled oracle parity, twice on one workspace (the arrival counters and
    the unit counter must be re-armed by the kernel itself), and the same result as the
    default split merge up to fp32 summation order."""
    monkeypatch.setenv("BKV_FUSED_MERGE", "1")
    o1 = _full_size(cfg, tp, 0, mode="step", pdl=True, seed=3, repeat=2)
    monkeypatch.setenv("BKV_FUSED_MERGE", "0")
    o0 = _full_size(cfg, tp, 0, mode="step", pdl=True, seed=3)
    assert (o0.float() - o1.float()).abs().max().item() <= 2e-2


@pytest.mark.parametrize("L0,bs,rt", [(8192, 32, 0.25), (8192, 16, 1.0), (512, 16, 0.0), (2048, 32, 0.75)])
def test_sweep_config_sampled_parity(L0, bs, rt):
    """BASELINE configs[4]: Llama-2-70B shape, context sweep 512-8K, block 16/32, RT:BE mix
    (TP8 shard: 1 kv head / 8 q heads), full batch 256, sampled requests vs the oracle."""
    from synth.workload import sweep_shape
    _full_size(sweep_shape(L0, bs, rt), tp=8, rank=3, seed=2, mode="step", pdl=True)


def _sampled_full_size(cfg, tp=1, rank=0, sample=6, seed=0, mode="attn", pdl=False, spare_blocks=3):
    """Kept for the one case whose host oracle pool would not fit (> 2^31-element pools): a
    full-size batch on the GPU, the oracle checks a sample of requests one by one.
    mode "attn": bkv_paged_decode_attention over the resident context; mode "step": the
    bench's launch configuration -- the fused decode step (bkv_decode_step, PDL) appending
    token L-1 of every request and attending over all L."""
    sh = CONFIGS[cfg] if isinstance(cfg, str) else cfg
    case = make_case(sh, seed, spare_blocks=spare_blocks)
    lay = case.layout
    kv_heads, q_heads = shard_heads(sh, tp, rank)
    Hl = len(kv_heads)
    pool = bkv.KVPool.empty(lay.num_blocks, Hl, sh.block_size, sh.head_dim, DEV)
    pool.k.zero_()
    pool.v.zero_()
    bt, dirs, lens = gpu_map(lay)
    resident = lay.lens - (1 if mode == "step" else 0)
    last_k, last_v = [], []
    for r0 in range(0, lay.batch, 32):   # generate on the GPU in request batches
        rs = range(r0, min(lay.batch, r0 + 32))
        kk, vv = zip(*[dense_kv_torch(case.seed, 0, r, int(lay.lens[r]), kv_heads, sh.head_dim,
                                      sh.num_kv_heads, DEV) for r in rs])
        last_k += [k[-1] for k in kk]
        last_v += [v[-1] for v in vv]
        kn = torch.cat([k[:resident[r]] for k, r in zip(kk, rs)])
        vn = torch.cat([v[:resident[r]] for v, r in zip(vv, rs)])
        cu = torch.tensor(np.concatenate([[0], np.cumsum(resident[list(rs)])]), dtype=torch.int32, device=DEV)
        sub_bt = bt[r0:r0 + len(rs)].contiguous()
        sub_dirs = dirs[r0:r0 + len(rs)].contiguous()
        bkv.kv_append(pool, sub_bt, sub_dirs, torch.zeros(len(rs), dtype=torch.int32, device=DEV), cu, kn, vn)
    q = torch.stack([q_torch(case.seed, 0, r, q_heads, sh.head_dim, DEV) for r in range(lay.batch)])
    if mode == "step":
        o = bkv.decode_step(pool, bt, dirs, lens, torch.stack(last_k).contiguous(),
                            torch.stack(last_v).contiguous(), q, pdl=pdl)
    else:
        o = bkv.paged_decode_attention(pool, bt, dirs, lens, q, pdl=pdl)
    torch.cuda.synchronize()
    # oracle on a sample of requests (longest, shortest, shared tails, random)
    rng = np.random.default_rng(seed + 100)
    order = np.argsort(lay.lens)
    pick = sorted(set([int(order[0]), int(order[-1])] + rng.choice(lay.batch, sample - 2, replace=False).tolist()))
    from synth import dense_kv_np, q_np
    for r in pick:
        L = int(lay.lens[r])
        k, v = dense_kv_np(case.seed, 0, r, L, kv_heads, sh.head_dim, sh.num_kv_heads)
        sub = build_layout([L], [bool(lay.is_be[r])], sh.block_size, rng, spare_blocks=1)
        K, V = oracle.new_pool(sub.num_blocks, Hl, sh.block_size, sh.head_dim, BF16_NAN)
        oracle.append(K, V, sub.block_tables, sub.dirs, np.zeros(1, np.int32), np.array([0, L], np.int32), k, v)
        qr = q_np(case.seed, 0, r, q_heads, sh.head_dim)[None]
        ref = oracle.attention(K, V, sub.block_tables, sub.dirs, sub.lens, qr, default_scale(sh.head_dim))
        check_close(o[r:r + 1], ref, f"{sh.name} r{r} L{L}")
    return o


def test_int64_offsets_tp1_8k_pool():
    """Llama-70B TP1 at 8K contexts: the pool holds > 2^31 elements per tensor, so every
    kernel's block/head/slot offsets must be 64-bit (sampled requests vs the oracle)."""
    from synth.workload import sweep_shape
    sh = sweep_shape(8192, 16, 0.5)
    lay = make_case(sh, 5, spare_blocks=4000).layout
    assert int(lay.block_tables.max()) * sh.num_kv_heads * sh.block_size * sh.head_dim > 2 ** 31
    _sampled_full_size(sh, tp=1, rank=0, sample=3, seed=5, mode="step", pdl=True, spare_blocks=4000)


def test_max_batch_2048():
    """num_seqs at the ABI maximum (2048): the in-kernel plan arrays are full."""
    sh = Shape("maxb", 4, 2, 64, 16, 2048, 0.5, "uniform", 96, 1, 1, uniform_max=96)
    _full_size(sh, 1, 0, seed=3, mode="step")
    _full_size(sh, 1, 0, seed=4, mode="attn")


# ---------------------------------------------------------------- ABI errors
def test_abi_argument_errors():
    pool = bkv.KVPool.empty(4, 1, 16, 96, DEV)   # head_dim 96 unsupported
    bt = torch.zeros(1, 1, dtype=torch.int32, device=DEV)
    dirs = torch.zeros(1, dtype=torch.uint8, device=DEV)
    lens = torch.ones(1, dtype=torch.int32, device=DEV)
    with pytest.raises(bkv.BkvError, match="head_dim 96"):
        bkv.paged_decode_attention(pool, bt, dirs, lens, torch.zeros(1, 1, 96, dtype=torch.bfloat16, device=DEV))
    pool = bkv.KVPool.empty(4, 2, 16, 64, DEV)
    with pytest.raises(bkv.BkvError, match="multiple"):
        bkv.paged_decode_attention(pool, bt, dirs, lens, torch.zeros(1, 3, 64, dtype=torch.bfloat16, device=DEV))
    small = torch.zeros(1024, dtype=torch.uint8, device=DEV)
    with pytest.raises(bkv.BkvError, match="WORKSPACE"):
        bkv.paged_decode_attention(pool, bt, dirs, lens, torch.zeros(1, 2, 64, dtype=torch.bfloat16, device=DEV), ws=small)


def test_pdl_launch_after_append_matches():
    """BKV_FLAG_PDL: attention launched right behind the kv_append that wrote the
    pool (programmatic dependent launch) gives bitwise the same output."""
    sh = Shape("pdl", 16, 2, 128, 16, 24, 0.5, "uniform", 600, 1, 1, uniform_max=600)
    case = make_case(sh, 31)
    lay = case.layout
    ks, vs, q = dense_case(case)
    before = (lay.lens - 1).astype(np.int32)
    B = lay.batch
    outs = []
    for pdl in (False, True):
        Kp, Vp = oracle.new_pool(lay.num_blocks, 2, 16, 128, BF16_NAN)
        kn, vn, cu = ragged(ks, vs, before, np.zeros(B, np.int32))
        oracle.append(Kp, Vp, lay.block_tables, lay.dirs, np.zeros(B, np.int32), cu, kn, vn)
        pool = bkv.KVPool(t_u16(Kp), t_u16(Vp))
        bt, dirs, lens = gpu_map(lay)
        kd, vd, cud = ragged(ks, vs, lay.lens, before)
        for _ in range(3):   # append then attention, back to back on one stream
            bkv.kv_append(pool, bt, dirs, torch.from_numpy(before).to(DEV), torch.from_numpy(cud).to(DEV),
                          t_u16(kd), t_u16(vd))
            o = bkv.paged_decode_attention(pool, bt, dirs, lens, t_u16(q), pdl=pdl)
        torch.cuda.synchronize()
        outs.append(o)
    assert torch.equal(outs[0].view(torch.int16), outs[1].view(torch.int16))
    K, V, _ = oracle_pool(case, ks, vs, 2)
    ref = oracle.attention(K, V, lay.block_tables, lay.dirs, lay.lens, q, default_scale(128))
    check_close(outs[1], ref, "pdl")


def test_mha_cuda_core_kernel_parity(monkeypatch):
    """g = 1 runs on the tensor-core kernel by default; the CUDA-core (FFMA2)
    kernel stays selectable (BKV_MHA_CUDA_CORES=1) and must agree with the oracle
    and, within 2x tolerance, with the tensor-core kernel."""
    monkeypatch.setenv("BKV_MHA_CUDA_CORES", "1")
    for cfg, seed in (("tiny", 40), ("tiny", 41)):
        case = make_case(cfg, seed)
        o_cc, ref, (ks, vs, q, pool) = _run_case(case)
        check_close(o_cc, ref, f"cuda-core {cfg}")
        lay = case.layout
        bt, dirs, lens = gpu_map(lay)
        monkeypatch.delenv("BKV_MHA_CUDA_CORES")
        o_tc = bkv.paged_decode_attention(pool, bt, dirs, lens, t_u16(q))
        torch.cuda.synchronize()
        check_close(o_tc, ref, f"tensor-core {cfg}")
        assert (o_cc.float() - o_tc.float()).abs().max().item() <= 2 * MAX_ABS
        monkeypatch.setenv("BKV_MHA_CUDA_CORES", "1")
    sh = Shape("cc", 5, 5, 128, 32, 20, 0.5, "uniform", 900, 1, 1, uniform_max=900)
    o, ref, _ = _run_case(make_case(sh, 42))
    check_close(o, ref, "cuda-core d128 bs32")


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("streamk", ["0", "2"])
def test_random_geometry_fuzz(seed, streamk, monkeypatch):
    """Seeded random geometries (group size, head_dim, block size, batch, lengths including
    empty contexts, RT/BE mix), both split plans, against the oracle."""
    monkeypatch.setenv("BKV_STREAMK", streamk)
    rng = np.random.default_rng(1000 + seed)
    hkv = int(rng.choice([1, 2, 4]))
    g = int(rng.choice([1, 2, 4, 8, 16]))
    d = int(rng.choice([64, 128]))
    bs = int(rng.choice([16, 32]))
    B = int(rng.integers(1, 48))
    lens = rng.integers(0, 1500, B)
    lens[rng.random(B) < 0.1] = 0
    is_be = (rng.random(B) < 0.5).tolist()
    sh = Shape("fuzz", hkv * g, hkv, d, bs, B, 0.5, "uniform", 1500, 1, 1)
    case = make_case(sh, seed, lens=lens.tolist(), is_be=is_be, q_scale_log2=int(rng.integers(0, 4)))
    o, ref, _ = _run_case(case)
    check_close(o, ref, f"fuzz{seed} g{g} hkv{hkv} d{d} bs{bs} B{B} sk{streamk}")
