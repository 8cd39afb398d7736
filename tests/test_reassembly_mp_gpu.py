"""Fused reassembly across PROCESSES: two ranks (gloo process group,
both on cuda:0 -- the only GPU a test box has) map each other's global output and flag
pad through torch CUDA IPC (tp.PeerReassembly), each runs the fused decode step on its
kv-head shard with bkv_decode_multi_out (its slice stored into BOTH global buffers) and
meets the other at bkv_peer_barrier.  Both global head-major outputs must be
bit-identical, equal the oracle within tolerance, and no barrier may time out.  On a
multi-GPU box the same code maps peer memory over NVLink.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2504_09590_b200 as bkv
        from paper_2504_09590_b200.tp import HeadShard, PeerReassembly
        from synth import make_case
        from tests._cases import dense_case
        from tests.test_fused_step import _prefilled, _step_rows
        from dataclasses import replace
        torch.cuda.set_device(0)
        case = make_case("tiny_gqa", seed)
        sh, lay = case.shape, case.layout
        shard = HeadShard(sh.num_q_heads, sh.num_kv_heads, world, rank)
        kvh, qh = list(shard.kv_heads), list(shard.q_heads)
        B, d = lay.batch, sh.head_dim
        ks, vs, qv = dense_case(case, kv_heads=kvh, q_heads=qh)
        sub = replace(case, shape=replace(sh, num_q_heads=len(qh), num_kv_heads=len(kvh)))
        K0, V0 = _prefilled(sub, ks, vs, (lay.lens - 1).astype(np.int32))
        g = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int16)).cuda().view(torch.bfloat16)
        pool = bkv.KVPool(g(K0), g(V0))
        kr, vr = _step_rows(ks, vs, lay.lens, len(kvh), d)
        bt = torch.from_numpy(lay.block_tables).cuda()
        dirs = torch.from_numpy(lay.dirs).cuda()
        lens = torch.from_numpy(lay.lens).cuda()
        re = PeerReassembly(shard, 2, B, d, torch.device("cuda", 0))
        for layer in range(2):     # two layers, two barriers (epochs 1, 2)
            bkv.decode_multi_out(pool if layer == 0 else bkv.KVPool(g(K0), g(V0)), bt, dirs, lens, g(qv),
                                 re.local_out(layer).permute(1, 0, 2), re.peer_outs(layer),
                                 k_new=g(kr), v_new=g(vr))
            re.barrier(timeout_ns=20_000_000_000)
        torch.cuda.synchronize()
        re.check()
        q.put((rank, re.glob.view(torch.int16).cpu().numpy()))
        dist.barrier()             # keep the buffers mapped until both ranks have read
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_process_p2p_reassembly_matches_oracle():
    import oracle
    from synth import make_case
    from tests._cases import dense_case, oracle_pool, default_scale
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 41, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert np.array_equal(got[0], got[1])
    case = make_case("tiny_gqa", 41)
    sh, lay = case.shape, case.layout
    ks, vs, qv = dense_case(case)
    K, V, _ = oracle_pool(case, ks, vs, sh.num_kv_heads)
    ref = oracle.attention(K, V, lay.block_tables, lay.dirs, lay.lens, qv, default_scale(sh.head_dim))
    for layer in range(2):
        o = got[0][layer].view(np.uint16)                       # [H_q][B][d] bf16 bits
        of = (o.astype(np.uint32) << 16).view(np.float32).astype(np.float64).transpose(1, 0, 2)
        err = np.abs(of - ref)
        assert err.max() <= 2e-2 and err.mean() <= 2e-3, (layer, err.max(), err.mean())
