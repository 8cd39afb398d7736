"""N > 1 path on CPU: world_size-2 gloo run of the head-sharded decode step.

Each rank owns half of the kv heads (and their q-head groups) of tiny_gqa,
draws the same GLOBAL values for its heads, runs the step with the CPU
oracle standing in for the CUDA kernels (append_fn / attn_fn), and the
all-gathered head-major output must equal the single-rank oracle bitwise.
This pins the sharding ranges, the per-rank value streams and the reassembly
order; the kernels themselves are covered by the GPU parity tests.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2504_09590_b200.tp import HeadShard, decode_step, gather_heads
from synth import make_case, dense_kv_np, q_np
from synth.values import BF16_NAN


class _HostPool:
    def __init__(self, K, V):
        self.K, self.V = K, V


def _append(pool, bt, dirs, before, cu, k_new, v_new):
    oracle.append(pool.K, pool.V, bt.numpy(), dirs.numpy(), before.numpy(), cu.numpy(),
                  k_new.numpy(), v_new.numpy())


def _attn_factory(lens_np, bt_np, dirs_np):
    def attn(pool, bt, dirs, lens, q_local, scale, out=None, max_seq_len=None, ws=None):
        o = oracle.attention(pool.K, pool.V, bt_np, dirs_np, lens_np, q_local.numpy(), scale)
        out.copy_(torch.from_numpy(o))
        return out
    return attn


def _expected(case):
    sh, lay = case.shape, case.layout
    H, d = sh.num_kv_heads, sh.head_dim
    K, V = oracle.new_pool(lay.num_blocks, H, sh.block_size, d, BF16_NAN)
    ks, vs = zip(*[dense_kv_np(case.seed, 0, r, int(lay.lens[r]), range(H), d, H) for r in range(lay.batch)])
    cu = np.concatenate([[0], np.cumsum(lay.lens)]).astype(np.int32)
    oracle.append(K, V, lay.block_tables, lay.dirs, np.zeros(lay.batch, np.int32), cu,
                  np.concatenate(ks), np.concatenate(vs))
    q = np.stack([q_np(case.seed, 0, r, range(sh.num_q_heads), d) for r in range(lay.batch)])
    out = oracle.attention(K, V, lay.block_tables, lay.dirs, lay.lens, q, 1.0 / np.sqrt(d))
    return out.transpose(1, 0, 2)   # head-major [H_q][B][d]


def _worker(rank, world, port, cfg, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        case = make_case(cfg, seed)
        sh, lay = case.shape, case.layout
        shard = HeadShard(sh.num_q_heads, sh.num_kv_heads, world, rank)
        kvh, qh = list(shard.kv_heads), list(shard.q_heads)
        d, B = sh.head_dim, lay.batch
        K, V = oracle.new_pool(lay.num_blocks, len(kvh), sh.block_size, d, BF16_NAN)
        ks, vs = zip(*[dense_kv_np(case.seed, 0, r, int(lay.lens[r]), kvh, d, sh.num_kv_heads) for r in range(B)])
        before = (lay.lens - 1).astype(np.int32)
        cu0 = np.concatenate([[0], np.cumsum(before)]).astype(np.int32)
        oracle.append(K, V, lay.block_tables, lay.dirs, np.zeros(B, np.int32), cu0,
                      np.concatenate([ks[r][:before[r]] for r in range(B)]),
                      np.concatenate([vs[r][:before[r]] for r in range(B)]))
        pool = _HostPool(K, V)
        k_new = torch.from_numpy(np.stack([ks[r][before[r]] for r in range(B)]))
        v_new = torch.from_numpy(np.stack([vs[r][before[r]] for r in range(B)]))
        q_glob = torch.from_numpy(np.stack([q_np(case.seed, 0, r, range(sh.num_q_heads), d) for r in range(B)]))
        q_loc = shard.local_q(q_glob)
        assert np.array_equal(q_loc.numpy(), np.stack([q_np(case.seed, 0, r, qh, d) for r in range(B)]))
        out_loc = torch.zeros((len(qh), B, d), dtype=torch.float64)
        out = decode_step(shard, pool, torch.from_numpy(lay.block_tables), torch.from_numpy(lay.dirs),
                          torch.from_numpy(before), torch.arange(B + 1, dtype=torch.int32), k_new, v_new,
                          torch.from_numpy(lay.lens), q_loc, out_loc, 1.0 / np.sqrt(d),
                          append_fn=_append, attn_fn=_attn_factory(lay.lens, lay.block_tables, lay.dirs))
        if rank == 0:
            q.put(out.numpy())
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("cfg,seed", [("tiny_gqa", 3), ("tiny", 4)])
def test_head_sharded_step_world2_matches_single_rank(cfg, seed):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cfg, seed, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    exp = _expected(make_case(cfg, seed))
    assert got.shape == exp.shape
    assert np.array_equal(got, exp)


def test_shard_ranges():
    s = [HeadShard(64, 8, 8, r) for r in range(8)]
    assert [list(x.kv_heads) for x in s] == [[r] for r in range(8)]
    assert [x.q_heads.start for x in s] == [8 * r for r in range(8)]
    s = HeadShard(40, 40, 2, 1)
    assert list(s.kv_heads) == list(range(20, 40)) and list(s.q_heads) == list(range(20, 40))
    with pytest.raises(ValueError):
        HeadShard(56, 56, 3, 0)
