"""Token-sharded data parallelism, host logic on CPU with gloo (world_size 2).

SURVEY.md §8(e): each rank quantizes and multiplies its token shard locally;
the only exchange is the fp32 dW all-reduce.  Each shard is an independent
tensor (own amax / scale32, own seeds), so the reference for the all-reduced
dW is sum_r backward(forward(X_r, W), E_r, seeds_r).dW computed by the oracle.
These tests run the oracle per rank (CPU), all-reduce through torch.distributed
(gloo, 127.0.0.1) and check the exchange reproduces that sum exactly, plus the
bench's per-rank seed derivation and shard bookkeeping.
"""

import os
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _shard_inputs(rank, tokens=128, din=128, dout=128):
    rng = np.random.default_rng(1000 + rank)
    x = rng.standard_normal((tokens, din)).astype(np.float32)
    e = (1e-2 * rng.standard_normal((tokens, dout))).astype(np.float32)
    w = (np.random.default_rng(7).standard_normal((dout, din)) / 16).astype(np.float32)   # replicated
    return x, w, e


def _seeds(rank, step):
    from oracle import nvfp4_oracle as O
    return O.SeedPair(O.derive_stream(1, step, rank), O.derive_stream(2, step, rank))


def _worker(rank, world, port, out_q):
    sys.path.insert(0, ROOT)
    from oracle import nvfp4_oracle as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    x, w, e = _shard_inputs(rank)
    _, tape = O.forward(x, w)
    dx, dw = O.backward(tape, e, _seeds(rank, 3), posthoc=True)
    t = torch.from_numpy(dw.astype(np.float32))
    dist.all_reduce(t)                       # the only collective of the layer
    g = [torch.zeros(1) for _ in range(world)]
    dist.all_gather(g, torch.tensor([float(dx.shape[0])]))
    if rank == 0:
        out_q.put((t.numpy(), [float(v) for v in g]))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_token_sharded_wgrad_allreduce():
    world = 2
    port = 29500 + (os.getpid() % 1000)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    dw, rows = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    sys.path.insert(0, ROOT)
    from oracle import nvfp4_oracle as O
    ref = np.zeros_like(dw, dtype=np.float64)
    for r in range(world):
        x, w, e = _shard_inputs(r)
        _, tape = O.forward(x, w)
        ref += O.backward(tape, e, _seeds(r, 3), posthoc=True)[1]
    np.testing.assert_allclose(dw, ref.astype(np.float32), rtol=1e-6, atol=1e-9)
    assert rows == [128.0, 128.0]


def test_rank_seeds_are_distinct_streams():
    s0, s1 = _seeds(0, 5), _seeds(1, 5)
    assert s0 != s1 and s0.rht != s1.rht and s0.sr != s1.sr
    assert _seeds(0, 5) == s0                # deterministic per (rank, step)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_weak_scaling_bookkeeping(world):
    """bench.py's value = flops over all ranks / max-rank time (weak scaling)."""
    sys.path.insert(0, ROOT)
    import bench
    per_gpu = bench.flops(bench.TOKENS)
    assert per_gpu == sum(6.0 * bench.TOKENS * i * o for _, i, o in bench.PROJECTIONS)
    assert bench.TOKENS % 128 == 0 and (65536 // max(world, 1)) % 128 == 0
