"""Two-rank NCCL run of the token-sharded step on real GPUs.

Each rank runs ShardedLinearStep with the CUDA layer on its token shard; the
all-reduced dW must equal the sum of the ranks' local dW (each recomputed
deterministically with the same per-rank seeds and gathered).  Skips unless two
GPUs are visible (the round-end box has one; the 8-GPU scaling runs use bench.py).
"""

import os
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, out_q, reduce="nccl"):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import paper_2601_22813_b200 as q2
    from paper_2601_22813_b200.parallel import ShardedLinearStep, shard_rows
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    g = torch.Generator(device=dev).manual_seed(3)
    X = torch.randn(1024, 256, device=dev, generator=g).bfloat16()
    W = (torch.randn(384, 256, device=dev, generator=g) / 16).bfloat16()
    E = (1e-2 * torch.randn(1024, 384, device=dev, generator=g)).bfloat16()
    sl = shard_rows(1024, rank, world)
    if reduce == "multimem":
        from paper_2601_22813_b200.parallel import MulticastReducer
        if not MulticastReducer.available():
            if rank == 0:
                out_q.put("skip")
            dist.barrier()
            dist.destroy_process_group()
            return
    runner = ShardedLinearStep(q2.LayerConfig(), rank=rank, world=world, reduce=reduce)
    (_, _, dw), = runner.step([(X[sl], W, E[sl])], 4)
    y, tape = q2.forward(X[sl], W, q2.LayerConfig(), out_dtype=torch.bfloat16)
    local = q2.backward(tape, E[sl], runner.seeds(4), dx_dtype=torch.bfloat16).dW
    parts = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(parts, local)
    # two ranks: a + b is order-free, so the switch's sum equals NCCL's bit for bit
    ok = torch.equal(dw, sum(parts[1:], parts[0]))
    if rank == 0:
        out_q.put(bool(ok))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("reduce", ["nccl", "multimem"])
def test_two_rank_nccl_sharded_step(reduce):
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, reduce)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=600)
    if ok == "skip":
        for p in procs:
            p.join(timeout=120)
        pytest.skip("no NVLS multicast on this pair")
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert ok
