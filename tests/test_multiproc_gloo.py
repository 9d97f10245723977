"""Token-sharded data parallelism, world_size 2 on CPU with gloo.

SURVEY.md §8(e): each rank quantizes and multiplies its token shard locally; the
only exchange is the fp32 dW all-reduce.  These tests run the PRODUCT's step driver
(paper_2601_22813_b200.parallel.ShardedLinearStep: shard bookkeeping, per-rank
seeds, async dW all-reduce per projection, wait at the end of the step) under
gloo on 127.0.0.1, with the CPU oracle injected as the per-shard linear (the
CUDA kernels need a GPU; their per-shard parity is the -m gpu suite).  The
all-reduced dW must equal sum_r backward(forward(X_r, W), E_r, seeds_r).dW.
"""

import os
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHAPES = ((128, 256), (256, 128))          # (in, out) of two projections
TOKENS = 256                               # global tokens, split over the ranks


def _global_inputs():
    rng = np.random.default_rng(1000)
    data = []
    for din, dout in SHAPES:
        x = rng.standard_normal((TOKENS, din)).astype(np.float32)
        w = (rng.standard_normal((dout, din)) / 16).astype(np.float32)       # replicated
        e = (1e-2 * rng.standard_normal((TOKENS, dout))).astype(np.float32)
        data.append((x, w, e))
    return data


def _oracle_linear(posthoc):
    from oracle import nvfp4_oracle as O

    def fwd(x, w):
        y, tape = O.forward(x.numpy(), w.numpy())
        return torch.from_numpy(y), tape

    def bwd(tape, e, seeds):
        dx, dw = O.backward(tape, e.numpy(), O.SeedPair(seeds.rht, seeds.sr), posthoc=posthoc)
        return torch.from_numpy(dx), torch.from_numpy(dw.astype(np.float32))
    return fwd, bwd


def _worker(rank, world, port, out_q):
    sys.path.insert(0, ROOT)
    from paper_2601_22813_b200.parallel import ShardedLinearStep, shard_rows
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sl = shard_rows(TOKENS, rank, world)
    data = [(torch.from_numpy(x[sl]), torch.from_numpy(w), torch.from_numpy(e[sl])) for x, w, e in _global_inputs()]
    fwd, bwd = _oracle_linear(posthoc=True)
    runner = ShardedLinearStep(rank=rank, world=world, seed=(1, 2), linear_fwd=fwd, linear_bwd=bwd)
    out = runner.step(data, 3)
    if rank == 0:
        out_q.put([dw.numpy() for _, _, dw in out] + [[int(y.shape[0]) for y, _, _ in out]])
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_sharded_step_allreduces_wgrad():
    world = 2
    port = 29500 + (os.getpid() % 1000)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    sys.path.insert(0, ROOT)
    from oracle import nvfp4_oracle as O
    from paper_2601_22813_b200.parallel import shard_rows, step_seeds
    rows = got.pop()
    assert rows == [TOKENS // world] * len(SHAPES)
    for j, (x, w, e) in enumerate(_global_inputs()):
        ref = np.zeros((w.shape[0], w.shape[1]), np.float64)
        for r in range(world):
            sl = shard_rows(TOKENS, r, world)
            s = step_seeds((1, 2), 3, r)
            _, tape = O.forward(x[sl], w)
            ref += O.backward(tape, e[sl], O.SeedPair(s.rht, s.sr), posthoc=True)[1].astype(np.float32)
        np.testing.assert_allclose(got[j], ref.astype(np.float32), rtol=1e-6, atol=1e-9)


def test_step_seeds_distinct_per_rank_and_step():
    sys.path.insert(0, ROOT)
    from paper_2601_22813_b200.parallel import step_seeds
    from paper_2601_22813_b200.rht import derive_stream
    s0, s1 = step_seeds((1, 2), 5, 0), step_seeds((1, 2), 5, 1)
    assert s0 != s1 and s0.rht != s1.rht and s0.sr != s1.sr
    assert step_seeds((1, 2), 5, 0) == s0 != step_seeds((1, 2), 6, 0)
    assert s0.rht == derive_stream(1, 5, 0) and s0.sr == derive_stream(2, 5, 0)


def test_shard_rows():
    sys.path.insert(0, ROOT)
    from paper_2601_22813_b200.parallel import shard_rows
    assert [shard_rows(65536, r, 4) for r in range(4)] == [slice(i * 16384, (i + 1) * 16384) for i in range(4)]
    with pytest.raises(ValueError):
        shard_rows(100, 0, 3)
    with pytest.raises(ValueError):
        shard_rows(128, 2, 2)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_weak_scaling_bookkeeping(world):
    """bench.py's value = flops over all ranks / max-rank time (weak scaling)."""
    sys.path.insert(0, ROOT)
    import bench
    per_gpu = bench.flops(bench.TOKENS)
    assert per_gpu == sum(6.0 * bench.TOKENS * i * o for _, i, o in bench.PROJECTIONS)
    assert bench.TOKENS % 128 == 0 and (65536 // max(world, 1)) % 128 == 0


def test_reducer_layout():
    from paper_2601_22813_b200.parallel import reducer_layout
    offs, n = reducer_layout([(6144, 2048), (2048, 2048), (3, 5)])
    assert offs == [0, 6144 * 2048, 6144 * 2048 + 2048 * 2048]
    assert n == offs[-1] + 64 and all(o % 64 == 0 for o in offs)
    with pytest.raises(ValueError):
        reducer_layout([(0, 4)])


def test_sharded_step_rejects_unknown_reduce():
    from paper_2601_22813_b200.parallel import ShardedLinearStep
    s = ShardedLinearStep(linear_fwd=lambda X, W: (X, None), linear_bwd=lambda t, E, s: (E, E), reduce="bogus")
    with pytest.raises(ValueError):
        s.step([(1, 2, 3)], 0)


class _FakeReducer:
    """Stands in for MulticastReducer on CPU: records the protocol calls."""

    def __init__(self, shapes):
        from paper_2601_22813_b200.parallel import reducer_layout
        self.shapes = [tuple(s) for s in shapes]
        self.offsets, _ = reducer_layout(self.shapes)
        self.mc_base = 1 << 40
        self.log = []
        import numpy as np
        self.views = [np.zeros(sh) for sh in self.shapes]

    def target(self, i):
        from paper_2601_22813_b200.parallel import MulticastReducer
        return MulticastReducer.target(self, i)          # the real address arithmetic

    def begin(self):
        self.log.append("begin")

    def finish(self):
        self.log.append("finish")


def test_sharded_step_multimem_protocol():
    """reduce="multimem": one begin() before the first wgrad, every backward gets its
    projection's dW slot and multicast address (base + 4 B x float offset), one finish()
    after the last, and no NCCL all-reduce is issued."""
    from paper_2601_22813_b200.parallel import ShardedLinearStep
    calls = []

    def bwd(tape, E, seeds, **kw):
        calls.append(kw)
        return E, kw["dw_out"]

    shapes = [(384, 256), (256, 256)]
    red = _FakeReducer(shapes)
    s = ShardedLinearStep(linear_fwd=lambda X, W: (X, None), linear_bwd=bwd, rank=0, world=2,
                          reduce="multimem", reducer=red)
    W = [type("W", (), {"shape": sh, "device": "cpu"})() for sh in shapes]
    out = s.step([(1, W[0], 2), (1, W[1], 3)], 0)
    assert red.log == ["begin", "finish"]
    assert [c["dw_accumulate"] for c in calls] == ["multimem", "multimem"]
    assert calls[0]["dw_multicast_ptr"] == (1 << 40)
    assert calls[1]["dw_multicast_ptr"] == (1 << 40) + 4 * 384 * 256
    assert out[1][2].shape == (256, 256)
