"""Serving-style robustness on the GPU (include/bkv.h conventions: stream-ordered,
graph-capturable, one workspace per stream, deterministic):
  * two batches decoded concurrently on two streams with two workspaces give
    bitwise the outputs of the same calls run one after the other;
  * a CUDA graph capturing the fused decode step + mixed prefill, replayed with
    new inputs copied into the captured buffers, matches eager calls bitwise.
"""
import numpy as np
import pytest
import torch

import paper_2504_09590_b200 as bkv
from synth import make_case
from tests._cases import dense_case
from tests.test_gpu_parity import DEV, gpu_map, gpu_pool_from_dense, t_u16

pytestmark = pytest.mark.gpu


def _setup(cfg, seed):
    case = make_case(cfg, seed)
    sh, lay = case.shape, case.layout
    ks, vs, q = dense_case(case)
    pool, _ = gpu_pool_from_dense(case, ks, vs, sh.num_kv_heads)
    bt, dirs, lens = gpu_map(lay)
    return case, pool, bt, dirs, lens, t_u16(q)


def test_two_streams_two_workspaces_match_serial():
    a = _setup("tiny_gqa", 51)
    b = _setup("llama70b", 52)   # full Llama batch shape on the full head set
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    ref = []
    for case, pool, bt, dirs, lens, q in (a, b):
        ref.append(bkv.paged_decode_attention(pool, bt, dirs, lens, q).clone())
    torch.cuda.synchronize()
    outs = []
    for (case, pool, bt, dirs, lens, q), s in ((a, s1), (b, s2)):
        with torch.cuda.stream(s):
            ws = bkv.workspace(q.shape[0], q.shape[1], pool.num_kv_heads, pool.head_dim, stream=s)
            outs.append(bkv.paged_decode_attention(pool, bt, dirs, lens, q, ws=ws, stream=s))
    torch.cuda.synchronize()
    for o, r in zip(outs, ref):
        assert torch.equal(o.view(torch.int16), r.view(torch.int16))


def test_graph_replay_with_new_inputs_matches_eager():
    case, pool, bt, dirs, lens, q = _setup("tiny_gqa", 53)
    sh, lay = case.shape, case.layout
    B, H, d = lay.batch, sh.num_kv_heads, sh.head_dim
    g = torch.Generator(device=DEV).manual_seed(7)
    kn = torch.randn(B, H, d, device=DEV, generator=g).to(torch.bfloat16)
    vn = torch.randn(B, H, d, device=DEV, generator=g).to(torch.bfloat16)
    qq = q.clone()
    out = torch.empty_like(q)
    ws = bkv.workspace(B, sh.num_q_heads, H, d)
    k_save, v_save = pool.k.clone(), pool.v.clone()
    # warm up, then capture the fused step on the captured buffers
    bkv.decode_step(pool, bt, dirs, lens, kn, vn, qq, out=out, ws=ws, pdl=True)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        bkv.decode_step(pool, bt, dirs, lens, kn, vn, qq, out=out, ws=ws, pdl=True)
    for it in range(3):
        new_q = torch.randn(q.shape, device=DEV, generator=g).to(torch.bfloat16)
        new_k = torch.randn(B, H, d, device=DEV, generator=g).to(torch.bfloat16)
        new_v = torch.randn(B, H, d, device=DEV, generator=g).to(torch.bfloat16)
        qq.copy_(new_q); kn.copy_(new_k); vn.copy_(new_v)
        pool.k.copy_(k_save); pool.v.copy_(v_save)
        graph.replay()
        torch.cuda.synchronize()
        got = out.clone()
        pool_after = pool.k.clone()
        pool.k.copy_(k_save); pool.v.copy_(v_save)
        ref = bkv.decode_step(pool, bt, dirs, lens, new_k, new_v, new_q)
        torch.cuda.synchronize()
        assert torch.equal(got.view(torch.int16), ref.view(torch.int16)), it
        assert torch.equal(pool_after.view(torch.int16), pool.k.view(torch.int16)), it


def test_prefill_graph_replay_matches_eager():
    from tests.test_prefill_oracle import make_q, query_counts
    case, pool, bt, dirs, lens, _ = _setup("tiny_gqa", 54)
    sh, lay = case.shape, case.layout
    n = query_counts(lay.lens, np.random.default_rng(54))
    qh, cu = make_q(case, n, sh.num_q_heads)
    q = t_u16(qh)
    cu_t = torch.from_numpy(cu).to(DEV)
    out = torch.empty_like(q)
    mq = int(n.max())
    bkv.paged_prefill_attention(pool, bt, dirs, lens, cu_t, q, max_q_len=mq, out=out)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        bkv.paged_prefill_attention(pool, bt, dirs, lens, cu_t, q, max_q_len=mq, out=out)
    graph.replay()
    torch.cuda.synchronize()
    ref = bkv.paged_prefill_attention(pool, bt, dirs, lens, cu_t, q, max_q_len=mq)
    torch.cuda.synchronize()
    assert torch.equal(out.view(torch.int16), ref.view(torch.int16))
