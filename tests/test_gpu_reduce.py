"""Reduction epilogues of the wgrad GEMM: ``accumulate="red"`` (atomic
adds, concurrent writers) and ``"multimem"`` (NVLS multicast: dW summed over ranks inside
the GEMM epilogue, the all-reduce after linear_graph.py:322-326 fused away).

On one GPU the "red" path is checked bit-exactly against the store / read-add-store
epilogues, and the multicast path runs on a one-rank symmetric-memory group when the
driver grants a multicast object (skipped otherwise); the two-rank sum is in
test_gpu_multigpu.py.
"""

import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from tests.families import make, to_bf16

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _q2():
    import paper_2601_22813_b200 as q2
    return q2


def _pair(m, n, k, seed):
    q2 = _q2()
    a = torch.from_numpy(make("normal", (m, k), seed)).cuda().bfloat16()
    b = torch.from_numpy(make("normal", (n, k), seed + 1)).cuda().bfloat16()
    return q2.quantize_rtn_46(a), q2.quantize_rtn_46(b)


@pytest.mark.parametrize("shape", [(256, 256, 512), (384, 640, 1024), (200, 136, 192)])
def test_gemm_red_matches_store(cuda, shape):
    q2 = _q2()
    qa, qb = _pair(*shape, seed=shape[0])
    d = q2.gemm(qa, qb)
    z = torch.zeros_like(d)
    q2.gemm(qa, qb, out=z, accumulate="red")
    assert torch.equal(z, d)                                # 0 + x == x (no subnormal products here)
    q2.gemm(qa, qb, out=z, accumulate="red")
    assert torch.equal(z, 2 * d)
    p = torch.randn_like(d)
    r, s = p.clone(), p.clone()
    q2.gemm(qa, qb, out=r, accumulate="red")
    q2.gemm(qa, qb, out=s, accumulate="add")
    assert torch.equal(r, s)                                # one fp32 add either way


def test_gemm_accumulate_argument_errors(cuda):
    q2 = _q2()
    qa, qb = _pair(256, 256, 256, 5)
    with pytest.raises(ValueError):
        q2.gemm(qa, qb, accumulate="red")                    # no out
    with pytest.raises(ValueError):
        q2.gemm(qa, qb, out=torch.zeros(256, 256, device="cuda"), accumulate="multimem")   # no address
    with pytest.raises(ValueError):
        q2.gemm(qa, qb, out=torch.zeros(256, 256, device="cuda", dtype=torch.bfloat16), accumulate="red")
    with pytest.raises(ValueError):
        q2.gemm(qa, qb, out=torch.zeros(256, 256, device="cuda"), accumulate="sum")


@pytest.mark.parametrize("posthoc", [False, True])
def test_backward_dw_out_modes(cuda, posthoc):
    """backward(..., dw_out=...) writes the same dW as the plain call, and "red" sums."""
    q2 = _q2()
    x = torch.from_numpy(make("normal", (512, 256), 1)).cuda().bfloat16()
    w = torch.from_numpy(to_bf16(make("normal", (384, 256), 2) / 16)).cuda().bfloat16()
    e = torch.from_numpy(to_bf16(1e-2 * make("normal", (512, 384), 3))).cuda().bfloat16()
    cfg = q2.LayerConfig(posthoc=posthoc)
    seeds = q2.SeedPair(11, 12)
    _, tape = q2.forward(x, w, cfg, out_dtype=torch.bfloat16)
    ref = q2.backward(tape, e, seeds, dx_dtype=torch.bfloat16)
    buf = torch.empty(384, 256, device="cuda")
    g = q2.backward(tape, e, seeds, dx_dtype=torch.bfloat16, dw_out=buf)
    assert g.dW.data_ptr() == buf.data_ptr()
    assert torch.equal(buf, ref.dW) and torch.equal(g.dX, ref.dX)
    buf.zero_()
    for _ in range(2):
        q2.backward(tape, e, seeds, dx_dtype=torch.bfloat16, dw_out=buf, dw_accumulate="red")
    torch.cuda.synchronize()
    assert torch.equal(buf, 2 * ref.dW)
    with pytest.raises(ValueError):
        q2.backward(tape, e, seeds, dw_out=torch.empty(256, 384, device="cuda"))


_ONE_GPU = r"""
import os, sys, torch
sys.path.insert(0, os.environ["Q2_ROOT"])
import paper_2601_22813_b200 as q2
from tests.families import make
from cuda.bindings import driver as d

import inspect
def ok(r):
    err = r[0] if isinstance(r, tuple) else r
    if err != d.CUresult.CUDA_SUCCESS:
        print("SKIP driver", err, "at line", inspect.currentframe().f_back.f_lineno); sys.exit(0)
    return r[1] if isinstance(r, tuple) and len(r) == 2 else r

torch.zeros(1, device="cuda")                      # primary context current
dev = ok(d.cuDeviceGet(0))
if not ok(d.cuDeviceGetAttribute(d.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)):
    print("SKIP device has no multicast support"); sys.exit(0)
M, N = 384, 640
prop = d.CUmulticastObjectProp()
prop.numDevices = 1
prop.handleTypes = d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
prop.size = 4 * M * N
gran = ok(d.cuMulticastGetGranularity(prop, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_MINIMUM))
size = -(-4 * M * N // gran) * gran
prop.size = size
mc = ok(d.cuMulticastCreate(prop))
ok(d.cuMulticastAddDevice(mc, dev))
ap = d.CUmemAllocationProp()
ap.type = d.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
ap.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
ap.location.id = 0
ap.requestedHandleTypes = d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
mem = ok(d.cuMemCreate(size, ap, 0))
ok(d.cuMulticastBindMem(mc, 0, mem, 0, size, 0))
acc = d.CUmemAccessDesc()
acc.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
acc.location.id = 0
acc.flags = d.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
uc = ok(d.cuMemAddressReserve(size, gran, 0, 0))
ok(d.cuMemMap(uc, size, 0, mem, 0))
ok(d.cuMemSetAccess(uc, size, [acc], 1))
mva = ok(d.cuMemAddressReserve(size, gran, 0, 0))
ok(d.cuMemMap(mva, size, 0, mc, 0))
ok(d.cuMemSetAccess(mva, size, [acc], 1))

class _Arr:
    __cuda_array_interface__ = {"shape": (M, N), "typestr": "<f4", "data": (int(uc), False), "version": 3}
view = torch.as_tensor(_Arr(), device="cuda")
a = torch.from_numpy(make("normal", (M, 1024), 7)).cuda().bfloat16()
b = torch.from_numpy(make("normal", (N, 1024), 8)).cuda().bfloat16()
qa, qb = q2.quantize_rtn_46(a), q2.quantize_rtn_46(b)
dd = q2.gemm(qa, qb)
view.zero_()
torch.cuda.synchronize()
q2.gemm(qa, qb, out=view, accumulate="multimem", multicast_ptr=int(mva))
q2.gemm(qa, qb, out=view, accumulate="multimem", multicast_ptr=int(mva))
torch.cuda.synchronize()
print("OK" if torch.equal(view, 2 * dd) else "MISMATCH %g" % (view - 2 * dd).abs().max().item())
"""


def test_multimem_one_gpu(cuda):
    """multimem.red.add.v4.f32 through a real one-device CUDA multicast object (driver API):
    the reductions land in the bound physical memory, bit-equal to 2 x the stored GEMM.
    (The round-2 gpurun boxes report MULTICAST_SUPPORTED = 1 but refuse cuMulticastCreate
    with INVALID_VALUE for every handle type: one GPU of an NVSwitch node in a container
    has no NVLS fabric -- the test then skips with the driver's answer.)"""
    env = dict(os.environ, Q2_ROOT=ROOT, PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", _ONE_GPU], env=env, cwd=ROOT, capture_output=True,
                       text=True, timeout=300)
    out = r.stdout.strip().splitlines()
    assert r.returncode == 0, r.stderr[-2000:]
    if out and out[-1].startswith("SKIP"):
        pytest.skip(out[-1])
    assert out and out[-1] == "OK", (r.stdout[-1000:], r.stderr[-1000:])


_ONE_RANK = r"""
import os, sys, torch, torch.distributed as dist
sys.path.insert(0, os.environ["Q2_ROOT"])
import paper_2601_22813_b200 as q2
from paper_2601_22813_b200.parallel import MulticastReducer
from tests.families import make
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=os.environ["Q2_PORT"])
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
try:
    red = MulticastReducer([(384, 640)], dev)
except Exception as exc:
    print("SKIP", type(exc).__name__, str(exc)[:200]); sys.exit(0)
a = torch.from_numpy(make("normal", (384, 1024), 7)).cuda().bfloat16()
b = torch.from_numpy(make("normal", (640, 1024), 8)).cuda().bfloat16()
qa, qb = q2.quantize_rtn_46(a), q2.quantize_rtn_46(b)
d = q2.gemm(qa, qb)
view, mc = red.target(0)
red.begin()
q2.gemm(qa, qb, out=view, accumulate="multimem", multicast_ptr=mc)
q2.gemm(qa, qb, out=view, accumulate="multimem", multicast_ptr=mc)
red.finish()
torch.cuda.synchronize()
print("OK" if torch.equal(view, 2 * d) else "MISMATCH %g" % (view - 2 * d).abs().max().item())
dist.destroy_process_group()
"""


def test_multimem_one_rank(cuda):
    """multimem.red.add through a real NVLS multicast object of a one-rank group."""
    env = dict(os.environ, Q2_ROOT=ROOT, Q2_PORT=str(29300 + os.getpid() % 500), PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", _ONE_RANK], env=env, cwd=ROOT, capture_output=True,
                       text=True, timeout=300)
    out = r.stdout.strip().splitlines()
    assert r.returncode == 0, r.stderr[-2000:]
    if out and out[-1].startswith("SKIP"):
        pytest.skip(out[-1])
    assert out and out[-1] == "OK", (r.stdout[-1000:], r.stderr[-1000:])
