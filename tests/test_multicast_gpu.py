"""NVLS multicast reassembly (PAPER.md P:759 moves these outputs
with NCCL): BKV_FLAG_PEER_MULTICAST stores every output row slice ONCE with
multimem.st to a multicast address, and the NVSwitch replicates it into every
buffer bound to the multicast object (every rank's global output on a TP box).

On one GPU the multicast object has one member: its physical buffer is bound,
mapped once through the multicast address (the kernels' target) and once
through a plain unicast address (what a rank reads).  Checked: after the
planned decode (both the decode-attention and the fused-step forms, and the
dynamically scheduled multi-out path) the unicast view of the bound buffer holds
exactly the bytes of the local output, which the oracle checks; the peer
barrier (with its alias fence) completes; the flag is rejected without exactly
one peer pointer.  Skipped where the device has no multicast support.
"""

import numpy as np
import pytest
import torch

import oracle
import paper_2504_09590_b200 as bkv
from synth import make_case

from tests._cases import dense_case, default_scale, oracle_pool
from tests.test_gpu_parity import DEV, check_close, gpu_map, gpu_pool_from_dense, t_u16

pytestmark = pytest.mark.gpu


def _drv():
    try:
        from cuda.bindings import driver
    except ImportError:   # older cuda-python layout
        from cuda import cuda as driver
    return driver


def _ok(res, what):
    err = res[0] if isinstance(res, tuple) else res
    drv = _drv()
    if err != drv.CUresult.CUDA_SUCCESS:
        raise RuntimeError(f"{what}: {err}")
    return res[1] if isinstance(res, tuple) and len(res) == 2 else res


class SingleDeviceMulticast:
    """A multicast object over ONE device with a bound physical buffer of >= nbytes,
    mapped at a multicast VA (mc) and a unicast VA (uc).  Plumbing for the test only."""

    def __init__(self, nbytes, dev=0):
        drv = _drv()
        torch.cuda.init()
        _ok(drv.cuInit(0), "cuInit")
        cudev = _ok(drv.cuDeviceGet(dev), "cuDeviceGet")
        sup = _ok(drv.cuDeviceGetAttribute(
            drv.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, cudev), "multicast attr")
        if not sup:
            pytest.skip("device reports no multicast (NVLS) support")
        prop = drv.CUmulticastObjectProp()
        prop.numDevices = 1
        prop.handleTypes = 0
        prop.size = nbytes
        gran = _ok(drv.cuMulticastGetGranularity(
            prop, drv.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED), "mc granularity")
        size = (nbytes + gran - 1) // gran * gran
        prop.size = size
        self.size = size
        res = drv.cuMulticastCreate(prop)
        if res[0] != drv.CUresult.CUDA_SUCCESS:
            pytest.skip(f"cuMulticastCreate failed: {res[0]}")
        self.mc_handle = res[1]
        _ok(drv.cuMulticastAddDevice(self.mc_handle, cudev), "cuMulticastAddDevice")
        aprop = drv.CUmemAllocationProp()
        aprop.type = drv.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        aprop.location.type = drv.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        aprop.location.id = dev
        self.phys = _ok(drv.cuMemCreate(size, aprop, 0), "cuMemCreate")
        _ok(drv.cuMulticastBindMem(self.mc_handle, 0, self.phys, 0, size, 0), "cuMulticastBindMem")
        acc = drv.CUmemAccessDesc()
        acc.location.type = drv.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        acc.location.id = dev
        acc.flags = drv.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        self.uc = int(_ok(drv.cuMemAddressReserve(size, gran, 0, 0), "reserve uc"))
        _ok(drv.cuMemMap(self.uc, size, 0, self.phys, 0), "map uc")
        _ok(drv.cuMemSetAccess(self.uc, size, [acc], 1), "access uc")
        self.mc = int(_ok(drv.cuMemAddressReserve(size, gran, 0, 0), "reserve mc"))
        _ok(drv.cuMemMap(self.mc, size, 0, self.mc_handle, 0), "map mc")
        _ok(drv.cuMemSetAccess(self.mc, size, [acc], 1), "access mc")
        _ok(drv.cuMemsetD8(self.uc, 0xAB, size), "memset uc")
        _ok(drv.cuCtxSynchronize(), "sync")

    def read(self, nbytes):
        drv = _drv()
        torch.cuda.synchronize()
        host = np.empty(nbytes, dtype=np.uint8)
        _ok(drv.cuMemcpyDtoH(host.ctypes.data, self.uc, nbytes), "cuMemcpyDtoH")
        return host

    def close(self):
        drv = _drv()
        torch.cuda.synchronize()
        drv.cuMemUnmap(self.mc, self.size)
        drv.cuMemUnmap(self.uc, self.size)
        drv.cuMemAddressFree(self.mc, self.size)
        drv.cuMemAddressFree(self.uc, self.size)
        drv.cuMulticastUnbind(self.mc_handle, 0, 0, self.size)
        drv.cuMemRelease(self.phys)
        drv.cuMemRelease(self.mc_handle)


def _case(cfg, seed):
    case = make_case(cfg, seed)
    sh, lay = case.shape, case.layout
    ks, vs, q = dense_case(case)
    K, V, _ = oracle_pool(case, ks, vs, sh.num_kv_heads)
    ref = oracle.attention(K, V, lay.block_tables, lay.dirs, lay.lens, q, default_scale(sh.head_dim))
    pool, _ = gpu_pool_from_dense(case, ks, vs, sh.num_kv_heads)
    return case, q, ref, pool


@pytest.mark.parametrize("cfg", ["tiny", "tiny_gqa", "llama70b"])
@pytest.mark.parametrize("path", ["planned", "multi_out"])
def test_multicast_reassembly_matches_local_output(cfg, path):
    case, q, ref, pool = _case(cfg, 41)
    sh, lay = case.shape, case.layout
    bt, dirs, lens = gpu_map(lay)
    out = torch.empty((lay.batch, sh.num_q_heads, sh.head_dim), dtype=torch.bfloat16, device=DEV)
    nbytes = out.numel() * 2
    mc = SingleDeviceMulticast(nbytes)
    try:
        if path == "planned":
            plan = bkv.decode_plan(lay.lens, lay.block_tables, lay.dirs, pool, sh.num_q_heads)
            bkv.decode_planned(pool, bt, dirs, lens, plan, t_u16(q), out=out, peer_outs=[mc.mc], multicast=True)
        else:
            bkv.decode_multi_out(pool, bt, dirs, lens, t_u16(q), out, [mc.mc], multicast=True)
        pads = torch.zeros((1,), dtype=torch.int32, device=DEV)
        counter = torch.zeros(1, dtype=torch.int32, device=DEV)
        err = torch.zeros(1, dtype=torch.int32, device=DEV)
        bkv.peer_barrier([pads.data_ptr()], 0, counter, err, 2_000_000_000)
        torch.cuda.synchronize()
        assert int(err.item()) == 0
        check_close(out, ref, cfg)
        got = mc.read(nbytes)
        assert np.array_equal(got, out.view(torch.uint8).cpu().numpy().ravel()), \
            "the multicast copy differs from the local output"
    finally:
        mc.close()


def test_multicast_fused_step_planned():
    """Fused decode step (append + attention) with multicast outputs: the bound buffer equals
    the local output bit for bit; the pool rows are appended as without multicast."""
    case, qd, _, pool = _case("tiny_gqa", 43)
    sh, lay = case.shape, case.layout
    bt, dirs, lens = gpu_map(lay)
    B, H, d = lay.batch, sh.num_kv_heads, sh.head_dim
    kn = torch.zeros((B, H, d), dtype=torch.bfloat16, device=DEV)
    vn = torch.zeros_like(kn)
    out = torch.empty((B, sh.num_q_heads, d), dtype=torch.bfloat16, device=DEV)
    out_ref = torch.empty_like(out)
    plan = bkv.decode_plan(lay.lens, lay.block_tables, lay.dirs, pool, sh.num_q_heads)
    # reference: the same fused step without multicast on a copy of the pool
    pool2 = bkv.KVPool(pool.k.clone(), pool.v.clone())
    bkv.decode_planned(pool2, bt, dirs, lens, plan, t_u16(qd), k_new=kn, v_new=vn, out=out_ref)
    mc = SingleDeviceMulticast(out.numel() * 2)
    try:
        bkv.decode_planned(pool, bt, dirs, lens, plan, t_u16(qd), k_new=kn, v_new=vn, out=out,
                           peer_outs=[mc.mc], multicast=True)
        torch.cuda.synchronize()
        assert torch.equal(out.view(torch.int16), out_ref.view(torch.int16))
        assert torch.equal(pool.k.view(torch.int16), pool2.k.view(torch.int16))
        assert torch.equal(pool.v.view(torch.int16), pool2.v.view(torch.int16))
        assert np.array_equal(mc.read(out.numel() * 2), out.view(torch.uint8).cpu().numpy().ravel())
    finally:
        mc.close()


def test_multicast_flag_needs_exactly_one_peer():
    case, q, ref, pool = _case("tiny", 44)
    sh, lay = case.shape, case.layout
    bt, dirs, lens = gpu_map(lay)
    out = torch.empty((lay.batch, sh.num_q_heads, sh.head_dim), dtype=torch.bfloat16, device=DEV)
    plan = bkv.decode_plan(lay.lens, lay.block_tables, lay.dirs, pool, sh.num_q_heads)
    with pytest.raises(bkv.BkvError, match="MULTICAST"):
        bkv.decode_planned(pool, bt, dirs, lens, plan, t_u16(q), out=out, multicast=True)
    with pytest.raises(bkv.BkvError, match="MULTICAST"):
        bkv.decode_multi_out(pool, bt, dirs, lens, t_u16(q), out, [out, out], multicast=True)
