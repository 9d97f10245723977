"""Token-sharded data parallelism for the Quartet II linear.

Rows of X and E are independent, so the layer shards on tokens: every rank holds
its own token shard and a replicated W, quantizes and multiplies locally (its own
amax / scale32, its own SR draws), and the only exchange is the fp32 dW sum.  Each
shard is an independent tensor exactly as if the reference were called on it
(linear_graph.py:243-333), so the parity target is the sum over ranks of
``backward(forward(X_r, W), E_r, seeds_r).dW``.

The dW all-reduce of one projection is issued asynchronously (NCCL over NVLink on
the GPU box, gloo in the CPU tests) and overlaps the next projection's work; the
step waits for all of them at its end.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence, Tuple

from .rht import SeedPair, derive_stream


def shard_rows(n_rows: int, rank: int, world: int) -> slice:
    """Contiguous token shard of rank ``rank`` (equal shards; n_rows % world == 0)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    if n_rows % world:
        raise ValueError(f"{n_rows} tokens do not split evenly over {world} ranks")
    per = n_rows // world
    return slice(rank * per, (rank + 1) * per)


def step_seeds(seed: Tuple[int, int], step: int, rank: int) -> SeedPair:
    """Per-rank, per-step seeds: derive_stream(seed, step, rank) for the rotation and
    the scale rounding (rht.py:78-86), so no two shards share SR draws."""
    return SeedPair(derive_stream(seed[0], step, rank), derive_stream(seed[1], step, rank))


@dataclass
class ShardedLinearStep:
    """One fwd+bwd step over a list of projections (X_r, W, E_r) on this rank.

    ``linear_fwd(X, W) -> (Y, tape)`` and ``linear_bwd(tape, E, seeds) -> (dX, dW)``
    default to the package's forward / backward with bf16 outputs; tests inject the
    CPU oracle to check the sharding, seeding and reduction logic under gloo.
    """

    cfg: object = None
    rank: int = 0
    world: int = 1
    group: object = None
    seed: Tuple[int, int] = (1, 2)
    linear_fwd: Optional[Callable] = None
    linear_bwd: Optional[Callable] = None
    last: List = field(default_factory=list)

    def __post_init__(self):
        if self.linear_fwd is None or self.linear_bwd is None:
            import torch

            from .linear_graph import LayerConfig, backward, forward
            cfg = self.cfg if self.cfg is not None else LayerConfig()
            if self.linear_fwd is None:
                self.linear_fwd = lambda X, W: forward(X, W, cfg, out_dtype=torch.bfloat16)
            if self.linear_bwd is None:
                def _bwd(tape, E, seeds):
                    g = backward(tape, E, seeds, dx_dtype=torch.bfloat16)
                    return g.dX, g.dW
                self.linear_bwd = _bwd

    def seeds(self, step: int) -> SeedPair:
        return step_seeds(self.seed, step, self.rank)

    def step(self, data: Sequence[tuple], i: int):
        """Run step ``i``; returns [(Y, dX, dW)] per projection, dW summed over ranks."""
        import torch.distributed as dist
        seeds = self.seeds(i)
        pending, out = [], []
        for X, W, E in data:
            y, tape = self.linear_fwd(X, W)
            dx, dw = self.linear_bwd(tape, E, seeds)
            if self.world > 1:                # the one exchange: dW, overlapping the next projection
                pending.append(dist.all_reduce(dw, group=self.group, async_op=True))
            out.append((y, dx, dw))
        for h in pending:
            h.wait()
        self.last = out
        return out
