"""Head-sharded tensor parallelism for the decode step.

The paper runs OPT-13B on 2, OPT-30B on 4 and Llama-70B on 8 GPUs with tensor
parallelism and moves tensors with NCCL.  For the
attention hot path that means: rank r owns kv heads [r*H/tp, (r+1)*H/tp) and
their query-head groups, keeps only those heads in its KV pool, runs
kv_append + decode attention on them, and -- only where the full output is
needed -- reassembles it with one all-gather.  Outputs are head-major
[H_q_local][B][d], so the rank-major concatenation produced by the all-gather
IS the global head-major [H_q][B][d]: no permute kernel.  Block tables,
direction tables and lengths are replicated (one host scheduler decision).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from .bkv import kv_append, paged_decode_attention


@dataclass(frozen=True)
class HeadShard:
    num_q_heads: int
    num_kv_heads: int
    tp: int
    rank: int

    def __post_init__(self):
        if self.num_kv_heads % self.tp:
            raise ValueError(f"{self.num_kv_heads} kv heads do not shard over tp={self.tp}")
        if self.num_q_heads % self.num_kv_heads:
            raise ValueError("num_q_heads must be a multiple of num_kv_heads")
        if not 0 <= self.rank < self.tp:
            raise ValueError("rank out of range")

    @property
    def group(self) -> int:
        return self.num_q_heads // self.num_kv_heads

    @property
    def kv_heads(self) -> range:   # global kv-head ids owned by this rank
        h = self.num_kv_heads // self.tp
        return range(self.rank * h, (self.rank + 1) * h)

    @property
    def q_heads(self) -> range:    # their query heads (groups stay intact, reading Q9)
        h = self.num_q_heads // self.tp
        return range(self.rank * h, (self.rank + 1) * h)

    def local_q(self, q_global: torch.Tensor) -> torch.Tensor:
        """[B][H_q][d] -> this rank's [B][H_q_local][d] view (no copy)."""
        return q_global[:, self.q_heads.start:self.q_heads.stop]

    def alloc_out(self, batch: int, head_dim: int, device, dtype=torch.bfloat16):
        """Head-major local output [H_q_local][B][d] (contiguous)."""
        return torch.empty((len(self.q_heads), batch, head_dim), dtype=dtype, device=device)


def gather_heads(out_local_hm: torch.Tensor, out_global_hm: torch.Tensor | None = None, group=None):
    """All-gather head-major shards into the global head-major [H_q][B][d]."""
    tp = dist.get_world_size(group)
    if out_global_hm is None:
        out_global_hm = torch.empty((out_local_hm.shape[0] * tp, *out_local_hm.shape[1:]),
                                    dtype=out_local_hm.dtype, device=out_local_hm.device)
    if tp == 1:
        out_global_hm.copy_(out_local_hm)
    elif dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out_global_hm, out_local_hm.contiguous(), group=group)
    else:   # gloo (CPU tests, single-GPU smoke runs): list all-gather on host copies, rank-major
        src = out_local_hm.detach().contiguous().cpu()
        parts = [torch.empty_like(src) for _ in range(tp)]
        dist.all_gather(parts, src, group=group)
        out_global_hm.copy_(torch.cat(parts, dim=0))
    return out_global_hm


def decode_step(shard: HeadShard, pool, block_tables, dirs, seq_lens_before, cu_new_tokens,
                k_new, v_new, seq_lens, q_local, out_local_hm, softmax_scale=None,
                out_global_hm=None, max_seq_len=None, ws=None, gather=True, group=None,
                append_fn=kv_append, attn_fn=paged_decode_attention):
    """One layer of one rank: append this step's tokens, attend, optionally all-gather.

    ``append_fn``/``attn_fn`` default to the CUDA kernels; tests substitute the
    CPU oracle to check the sharding and reassembly logic without a GPU.
    """
    append_fn(pool, block_tables, dirs, seq_lens_before, cu_new_tokens, k_new, v_new)
    attn_fn(pool, block_tables, dirs, seq_lens, q_local, softmax_scale,
            out=out_local_hm.permute(1, 0, 2), max_seq_len=max_seq_len, ws=ws)
    if gather and shard.tp > 1:
        return gather_heads(out_local_hm, out_global_hm, group)
    return out_local_hm


class PeerReassembly:
    """Fused reassembly over NVLink: every rank's decode kernels store its
    head slice straight into every peer's global head-major output, then one stream-ordered
    peer barrier publishes completion -- no separate all-gather.

    Plumbing only: each rank allocates its global output [n_layers][H_q][B][d] and a flag
    pad with torch, exports them with torch's CUDA IPC (``reduce_tensor``, the mechanism of
    torch.multiprocessing) through the process group, and maps the peers' buffers (P2P over
    NVLink between GPUs; also valid for several ranks on one GPU).  The stores and the
    barrier are libbkv kernels (bkv_decode_multi_out, bkv_peer_barrier).
    """

    def __init__(self, shard: HeadShard, n_layers: int, batch: int, head_dim: int, device, group=None):
        from torch.multiprocessing.reductions import reduce_tensor
        self.shard = shard
        hq, hl = shard.num_q_heads, len(shard.q_heads)
        self.glob = torch.zeros((n_layers, hq, batch, head_dim), dtype=torch.bfloat16, device=device)
        self.pads = torch.zeros((shard.tp,), dtype=torch.int32, device=device)
        torch.cuda.synchronize(device)
        mine = (reduce_tensor(self.glob), reduce_tensor(self.pads))
        allh = [None] * shard.tp
        dist.all_gather_object(allh, mine, group=group)
        self._peer_tensors = []   # keep the mapped peer tensors alive
        bases, pads = [], []
        for k, (hg, hp) in enumerate(allh):
            if k == shard.rank:
                g_k, p_k = self.glob, self.pads
            else:
                g_k, p_k = hg[0](*hg[1]), hp[0](*hp[1])
                self._peer_tensors += [g_k, p_k]
            bases.append(g_k.data_ptr())
            pads.append(p_k.data_ptr())
        esz = self.glob.element_size()
        self.layer_bytes = hq * batch * head_dim * esz
        self.slice_off = shard.rank * hl * batch * head_dim * esz
        self.peer_bases = [b for k, b in enumerate(bases) if k != shard.rank]
        self.pad_ptrs = pads
        self.counter = torch.zeros(1, dtype=torch.int32, device=device)
        self.err = torch.zeros(1, dtype=torch.int32, device=device)
        torch.cuda.synchronize(device)
        dist.barrier(group)

    def local_out(self, layer: int) -> torch.Tensor:
        """This rank's slice of its own global output, head-major [H_q_local][B][d]."""
        hl = len(self.shard.q_heads)
        return self.glob[layer, self.shard.rank * hl:(self.shard.rank + 1) * hl]

    def peer_outs(self, layer: int):
        return [b + layer * self.layer_bytes + self.slice_off for b in self.peer_bases]

    def barrier(self, timeout_ns: int = 5_000_000_000):
        from .bkv import peer_barrier
        peer_barrier(self.pad_ptrs, self.shard.rank, self.counter, self.err, timeout_ns)

    def check(self):
        """Raise if a peer barrier timed out (call outside timed regions)."""
        if int(self.err.item()) != 0:
            raise RuntimeError("bkv_peer_barrier timed out: a peer rank did not arrive")


class MulticastReassembly(PeerReassembly):
    """Fused reassembly through an NVLS multicast object (BKV_FLAG_PEER_MULTICAST):
    every rank's global output [n_layers][H_q][B][d] is bound to one multicast object, and
    the decode kernels store each row slice ONCE to the multicast address; the NVSwitch writes
    it into every rank's buffer (instead of n_peers separate NVLink stores).  Completion: the
    same peer barrier (its alias fence orders the multicast stores before the release).

    Plumbing only, through torch symmetric memory (allocation, handle exchange, multicast
    mapping): needs a CUDA process group on GPUs joined by NVSwitch with multicast support;
    raises if the runtime offers no multicast address.  Same interface as PeerReassembly,
    ``multicast = True`` tells the caller to pass BKV_FLAG_PEER_MULTICAST."""

    multicast = True

    def __init__(self, shard: HeadShard, n_layers: int, batch: int, head_dim: int, device, group=None):
        import torch.distributed._symmetric_memory as symm_mem
        self.shard = shard
        hq, hl = shard.num_q_heads, len(shard.q_heads)
        grp = group if group is not None else dist.group.WORLD
        gname = grp.group_name
        if hasattr(symm_mem, "enable_symm_mem_for_group"):
            symm_mem.enable_symm_mem_for_group(gname)
        self.glob = symm_mem.empty((n_layers, hq, batch, head_dim), dtype=torch.bfloat16, device=device)
        self.glob.zero_()
        self._hdl = symm_mem.rendezvous(self.glob, gname)
        mc = int(getattr(self._hdl, "multicast_ptr", 0) or 0)
        if mc == 0:
            raise RuntimeError("no NVLS multicast address for this group (needs NVSwitch multicast support)")
        self.pads = symm_mem.empty((shard.tp,), dtype=torch.int32, device=device)
        self.pads.zero_()
        self._hdl_pads = symm_mem.rendezvous(self.pads, gname)
        self.pad_ptrs = [int(x) for x in self._hdl_pads.buffer_ptrs]
        esz = self.glob.element_size()
        self.layer_bytes = hq * batch * head_dim * esz
        self.slice_off = shard.rank * hl * batch * head_dim * esz
        self.mc_base = mc
        self.counter = torch.zeros(1, dtype=torch.int32, device=device)
        self.err = torch.zeros(1, dtype=torch.int32, device=device)
        torch.cuda.synchronize(device)
        dist.barrier(grp)

    def peer_outs(self, layer: int):
        """ONE pointer: this rank's slice of layer `layer` in the multicast mapping."""
        return [self.mc_base + layer * self.layer_bytes + self.slice_off]
