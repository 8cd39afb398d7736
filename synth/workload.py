"""Seeded request-length and block-layout generator (host side, no method arithmetic).

Length recipe:
  * RT ShareGPT / LMSYS-Chat-1M: prompt and output lengths lognormal, fitted by
    moments to Table "Workload statistics":
      ShareGPT  prompt 222.76 +- 256.36, output 234.51 +- 268.50
      LMSYS     prompt  90.50 +- 148.52, output 237.04 +- 228.21
  * BE synthetic: prompt U[512, 1024], output U[32, 128] (moments P:750).
  * A decode snapshot of a request sits somewhere inside its generation:
    resident length L = prompt + U{1..output}, clamped to the model context.
Layout recipe (stand-in for FindBlock / FindPreemptBlock):
  * every request owns ceil(L/bs) block-table entries; all non-tail entries are
    full (reading Q6), the tail entry holds the remaining 1..bs tokens;
  * RT and BE tails are paired greedily into one shared physical block when
    their fills fit together ("one RT request and one BE request" per block);
  * physical block ids are a seeded random permutation of the pool.
The generator never computes a slot index: which slot a token lands in is the
method's business (oracle/ and the CUDA path each implement it on their own).
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace
import math

import numpy as np

RT, BE = 0, 1   # direction flag values: 0 = forward (RT), 1 = reversed (BE)  -- P:711


@dataclass(frozen=True)
class Shape:
    name: str
    num_q_heads: int
    num_kv_heads: int
    head_dim: int
    block_size: int
    batch: int
    rt_fraction: float
    rt_dist: str            # 'sharegpt' | 'lmsys' | 'uniform' | 'sweep'
    max_ctx: int
    n_layers: int
    default_tp: int
    uniform_max: int = 256  # for rt_dist == 'uniform'
    sweep_len: int = 0      # for rt_dist == 'sweep': L = L0 - U{0..bs-1}

    @property
    def group(self) -> int:
        return self.num_q_heads // self.num_kv_heads


CONFIGS = {
    # BASELINE.json configs[0]: 1 layer, 4 heads, d64, bs16, 8 requests (4 RT + 4 BE), ctx <= 256
    "tiny": Shape("tiny", 4, 4, 64, 16, 8, 0.5, "uniform", 256, 1, 1, uniform_max=256),
    # parity-only GQA variant: 8 Q / 2 KV heads, d128
    "tiny_gqa": Shape("tiny_gqa", 8, 2, 128, 16, 8, 0.5, "uniform", 256, 1, 1, uniform_max=256),
    # configs[1]: OPT-13B shape 40 x d128, ShareGPT, mixed batch 64, TP2 in the paper
    "opt13b": Shape("opt13b", 40, 40, 128, 16, 64, 0.5, "sharegpt", 2048, 40, 2),
    # configs[2]: OPT-30B shape 56 x d128, LMSYS, mixed batch 128, TP4
    "opt30b": Shape("opt30b", 56, 56, 128, 16, 128, 0.5, "lmsys", 2048, 48, 4),
    # configs[3]: Llama-2-70B shape 64 Q / 8 KV x d128 (GQA 8), ShareGPT, batch 256, TP8
    "llama70b": Shape("llama70b", 64, 8, 128, 16, 256, 0.5, "sharegpt", 4096, 80, 8),
}


def sweep_shape(L0: int, bs: int = 16, rt_fraction: float = 0.5) -> Shape:
    """configs[4]: RT:BE ratio and context sweep on the Llama-2-70B shape."""
    return Shape(f"sweep_L{L0}_bs{bs}_rt{rt_fraction:g}", 64, 8, 128, bs, 256, rt_fraction,
                 "sweep", max(L0, 8192), 80, 8, sweep_len=L0)


_MOMENTS = {  # (prompt mean, prompt std, output mean, output std) -- P:748-749
    "sharegpt": (222.76, 256.36, 234.51, 268.50),
    "lmsys": (90.50, 148.52, 237.04, 228.21),
}


def _lognormal(rng, mean, std, n):
    s2 = math.log(1.0 + (std / mean) ** 2)
    mu = math.log(mean) - s2 / 2.0
    return rng.lognormal(mu, math.sqrt(s2), n)


def draw_lengths(shape: Shape, rng: np.random.Generator):
    """Return (L int64[B] resident lengths incl. this step's token, is_be bool[B])."""
    B = shape.batch
    n_rt = int(round(B * shape.rt_fraction))
    is_be = np.zeros(B, dtype=bool)
    is_be[n_rt:] = True
    rng.shuffle(is_be)
    L = np.zeros(B, dtype=np.int64)
    if shape.rt_dist == "uniform":
        L[:] = rng.integers(1, shape.uniform_max + 1, B)
    elif shape.rt_dist == "sweep":
        L[:] = shape.sweep_len - rng.integers(0, shape.block_size, B)
    else:
        pm, ps, om, os_ = _MOMENTS[shape.rt_dist]
        nr = int((~is_be).sum())
        prompt = np.maximum(1, np.rint(_lognormal(rng, pm, ps, nr))).astype(np.int64)
        out = np.maximum(1, np.rint(_lognormal(rng, om, os_, nr))).astype(np.int64)
        gen = np.floor(rng.random(nr) * out).astype(np.int64) + 1          # U{1..output}
        L[~is_be] = prompt + gen
        nb = int(is_be.sum())
        bprompt = rng.integers(512, 1025, nb)
        bout = rng.integers(32, 129, nb)
        bgen = np.floor(rng.random(nb) * bout).astype(np.int64) + 1
        L[is_be] = bprompt + bgen
    L = np.clip(L, 1, shape.max_ctx)
    return L, is_be


@dataclass
class Layout:
    """Host-side block map for one batch (D2 block table + D3 direction table + D4 lengths)."""
    lens: np.ndarray              # int32 [B]  resident tokens incl. the one appended this step
    is_be: np.ndarray             # bool  [B]
    block_size: int
    block_tables: np.ndarray      # int32 [B][M], -1 padded
    dirs: np.ndarray              # uint8 [B][M] per-entry direction (0 RT fwd, 1 BE rev), 0 padded
    num_blocks: int               # pool capacity in blocks
    n_shared: int                 # number of physical blocks shared by an RT and a BE request
    fills: np.ndarray | None = None        # general map only (f3): uint8 [B][M] tokens per entry
    num_entries: np.ndarray | None = None  # general map only (f3): int32 [B] entries in use

    @property
    def batch(self) -> int:
        return int(self.lens.shape[0])

    @property
    def dirs_per_request(self) -> np.ndarray:
        return self.is_be.astype(np.uint8)

    def nblocks(self) -> np.ndarray:
        if self.num_entries is not None:
            return self.num_entries.astype(np.int64)
        return (self.lens + self.block_size - 1) // self.block_size

    @property
    def general(self) -> bool:
        return self.fills is not None


def build_layout(lens, is_be, block_size: int, rng: np.random.Generator, *,
                 share_tails: bool = True, spare_blocks: int = 0, max_blocks: int | None = None,
                 permute: bool = True) -> Layout:
    lens = np.asarray(lens, dtype=np.int64)
    is_be = np.asarray(is_be, dtype=bool)
    B = lens.shape[0]
    bs = block_size
    nb = np.where(lens > 0, (lens + bs - 1) // bs, 0)
    fill = np.where(lens > 0, lens - (nb - 1) * bs, 0)
    # greedy two-pointer pairing of RT tails (largest first) with BE tails (smallest first)
    pairs = []
    if share_tails:
        rt = sorted([r for r in range(B) if not is_be[r] and nb[r] > 0], key=lambda r: -fill[r])
        be = sorted([r for r in range(B) if is_be[r] and nb[r] > 0], key=lambda r: fill[r])
        j = 0
        for r in rt:
            if j < len(be) and fill[r] + fill[be[j]] <= bs:
                pairs.append((r, be[j]))
                j += 1
    tail_partner = {}
    for a, b in pairs:
        tail_partner[b] = a
    M = int(max_blocks if max_blocks is not None else max(1, int(nb.max()) if B else 1))
    assert M >= (int(nb.max()) if B else 0)
    logical = np.full((B, M), -1, dtype=np.int64)
    nxt = 0
    for r in range(B):
        for e in range(nb[r]):
            if e == nb[r] - 1 and r in tail_partner:
                continue                      # filled below from the RT partner's tail
            logical[r, e] = nxt
            nxt += 1
    for b, a in tail_partner.items():
        logical[b, nb[b] - 1] = logical[a, nb[a] - 1]
    num_blocks = nxt + int(spare_blocks)
    perm = rng.permutation(num_blocks) if permute else np.arange(num_blocks)
    bt = np.where(logical >= 0, perm[np.maximum(logical, 0)], -1).astype(np.int32)
    dirs = np.zeros((B, M), dtype=np.uint8)
    for r in range(B):
        dirs[r, :nb[r]] = BE if is_be[r] else RT
    return Layout(lens.astype(np.int32), is_be, bs, bt, dirs, max(num_blocks, 1), len(pairs))


def build_general_layout(lens, is_be, block_size: int, rng: np.random.Generator, *,
                         share_prob: float = 0.6, spare_blocks: int = 0, permute: bool = True,
                         order=None) -> Layout:
    """General map: any entry may be partly filled.

    Stand-in for FindBlock (a BE prefill goes to "the blocks with
    the maximum number of empty slots") and FindPreemptBlock (an
    RT request takes over a BE block "from the opposite end").  Requests are
    placed one after another (seeded random order).  Each takes blocks until
    its tokens are placed: with probability ``share_prob`` it reuses, among the
    blocks whose own-direction side is free and whose opposite side is in use,
    the one with the most empty slots, putting min(remaining, empty) tokens
    there; otherwise a fresh block takes min(remaining, bs).  The output is
    only WHICH block each entry names and HOW MANY tokens it holds -- never a
    slot index (that is the method's business).
    """
    lens = np.asarray(lens, dtype=np.int64)
    is_be = np.asarray(is_be, dtype=bool)
    B, bs = lens.shape[0], block_size
    used = [[0, 0]]  # per logical block: tokens of its forward / reversed owner (0 = side free)
    used.clear()
    entries = [[] for _ in range(B)]
    n_shared = 0
    order = rng.permutation(B) if order is None else np.asarray(order)
    for r in order:
        d = int(is_be[r])
        rem = int(lens[r])
        while rem > 0:
            blk = -1
            if rng.random() < share_prob:
                best = 0
                for b, u in enumerate(used):
                    empty = bs - u[0] - u[1]
                    if u[d] == 0 and u[1 - d] > 0 and empty > best:
                        best, blk = empty, b
            if blk < 0:
                used.append([0, 0])
                blk = len(used) - 1
            else:
                n_shared += 1
            n = min(rem, bs - used[blk][0] - used[blk][1])
            used[blk][d] = n
            entries[r].append((blk, n))
            rem -= n
    M = max(1, max((len(e) for e in entries), default=1))
    num_blocks = len(used) + int(spare_blocks)
    perm = rng.permutation(num_blocks) if permute else np.arange(num_blocks)
    bt = np.full((B, M), -1, dtype=np.int32)
    fills = np.zeros((B, M), dtype=np.uint8)
    dirs = np.zeros((B, M), dtype=np.uint8)
    nent = np.zeros(B, dtype=np.int32)
    for r in range(B):
        nent[r] = len(entries[r])
        for e, (blk, n) in enumerate(entries[r]):
            bt[r, e] = perm[blk]
            fills[r, e] = n
            dirs[r, e] = BE if is_be[r] else RT
    return Layout(lens.astype(np.int32), is_be, bs, bt, dirs, max(num_blocks, 1), n_shared,
                  fills=fills, num_entries=nent)


@dataclass
class Case:
    """One seeded batch: shape, layout and the value-stream seed."""
    shape: Shape
    layout: Layout
    seed: int
    q_scale_log2: int = 0
    layer: int = 0


def make_case(shape: Shape | str, seed: int = 0, *, lens=None, is_be=None, share_tails=True,
              spare_blocks: int = 3, q_scale_log2: int = 0, layer: int = 0,
              general: bool = False, share_prob: float = 0.6) -> Case:
    if isinstance(shape, str):
        shape = CONFIGS[shape]
    rng = np.random.default_rng(seed)
    if lens is None:
        lens, is_be2 = draw_lengths(shape, rng)
        if is_be is None:
            is_be = is_be2
    else:
        lens = np.asarray(lens, dtype=np.int64)
        if is_be is None:
            is_be = np.arange(len(lens)) % 2 == 1
        shape = replace(shape, batch=len(lens))
    if general:
        lay = build_general_layout(lens, is_be, shape.block_size, rng, share_prob=share_prob,
                                   spare_blocks=spare_blocks)
    else:
        lay = build_layout(lens, is_be, shape.block_size, rng, share_tails=share_tails,
                           spare_blocks=spare_blocks)
    return Case(shape, lay, seed, q_scale_log2, layer)


def shard_heads(shape: Shape, tp: int, rank: int):
    """Global (kv_heads, q_heads) owned by ``rank`` under head-sharded TP."""
    assert shape.num_kv_heads % tp == 0, "kv heads must divide by tp"
    hkv = shape.num_kv_heads // tp
    g = shape.group
    kv = list(range(rank * hkv, (rank + 1) * hkv))
    q = list(range(rank * hkv * g, (rank + 1) * hkv * g))
    return kv, q
