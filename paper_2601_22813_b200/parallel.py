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


def reducer_layout(shapes: Sequence[Tuple[int, int]], align: int = 64) -> Tuple[List[int], int]:
    """Float offsets of the per-projection dW buffers inside one symmetric allocation
    (each start aligned to ``align`` floats = 256 B, the GEMM's 16-byte rule with room)
    and the total float count."""
    offs, n = [], 0
    for r, c in shapes:
        if r <= 0 or c <= 0:
            raise ValueError(f"bad dW shape {(r, c)}")
        offs.append(n)
        n += -(-(r * c) // align) * align
    return offs, n


class MulticastReducer:
    """The dW all-reduce fused into the wgrad GEMM epilogue over NVLink SHARP (NVLS).

    One symmetric-memory fp32 allocation (torch.distributed._symmetric_memory) holds a dW
    buffer per projection on every rank; its NVLS multicast address goes to the GEMM
    (``accumulate="multimem"``), whose epilogue issues ``multimem.red.add.v4.f32`` so the
    NVSwitch adds each rank's tile into every rank's replica -- no separate collective and
    no second pass over dW (the reference sums dW after linear_graph.py:322-326; SURVEY
    §8(f)-3).  Protocol per step: ``begin()`` zeroes the local replicas and barriers (no
    rank reduces into a replica before its owner cleared it), the wgrad GEMMs run, and
    ``finish()`` barriers (every rank's reductions have landed; the GEMM ends with a
    ``fence.acq_rel.sys``).  The dW views are overwritten by the next ``begin()``.
    Summation order across ranks is the switch's, as with an NCCL all-reduce; reductions
    flush fp32 subnormals.
    """

    def __init__(self, shapes: Sequence[Tuple[int, int]], device, group=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem
        group = group if group is not None else dist.group.WORLD
        self.offsets, total = reducer_layout(shapes)
        self.shapes = [tuple(s) for s in shapes]
        name = group.group_name
        try:
            if not symm_mem.is_symm_mem_enabled_for_group(name):
                symm_mem.enable_symm_mem_for_group(name)
        except Exception:                                   # newer torch: always enabled
            pass
        self.buf = symm_mem.empty(total, dtype=torch.float32, device=device)
        self.hdl = symm_mem.rendezvous(self.buf, name)
        mc = int(getattr(self.hdl, "multicast_ptr", 0) or 0)
        if not mc:
            raise RuntimeError("NVLS multicast is not available on this group (needs NVSwitch, "
                               "CUDA multicast objects and world_size > 1)")
        base = int(self.hdl.buffer_ptrs[self.hdl.rank])
        self.mc_base = mc + (self.buf.data_ptr() - base)
        self.views = [self.buf[o:o + r * c].view(r, c) for o, (r, c) in zip(self.offsets, self.shapes)]

    @staticmethod
    def available(group=None) -> bool:
        """True when a multicast-capable symmetric allocation can be made on ``group``."""
        try:
            import torch
            import torch.distributed as dist
            if not dist.is_initialized() or dist.get_world_size(group) < 2 or not torch.cuda.is_available():
                return False
            MulticastReducer([(1, 64)], torch.device("cuda", torch.cuda.current_device()), group)
            return True
        except Exception:
            return False

    def target(self, i: int):
        """(dW view, its multicast address) of projection ``i``."""
        return self.views[i], self.mc_base + 4 * self.offsets[i]

    def begin(self) -> None:
        self.buf.zero_()
        self.hdl.barrier(channel=0)

    def finish(self) -> None:
        self.hdl.barrier(channel=0)


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
    reduce: str = "nccl"          # "nccl": async all-reduce per projection; "multimem": NVLS in the GEMM
    last: List = field(default_factory=list)
    reducer: object = None

    def __post_init__(self):
        if self.linear_fwd is None or self.linear_bwd is None:
            import torch

            from .linear_graph import LayerConfig, backward, forward
            cfg = self.cfg if self.cfg is not None else LayerConfig()
            if self.linear_fwd is None:
                self.linear_fwd = lambda X, W: forward(X, W, cfg, out_dtype=torch.bfloat16)
            if self.linear_bwd is None:
                def _bwd(tape, E, seeds, **kw):
                    g = backward(tape, E, seeds, dx_dtype=torch.bfloat16, **kw)
                    return g.dX, g.dW
                self.linear_bwd = _bwd

    def seeds(self, step: int) -> SeedPair:
        return step_seeds(self.seed, step, self.rank)

    def step(self, data: Sequence[tuple], i: int):
        """Run step ``i``; returns [(Y, dX, dW)] per projection, dW summed over ranks."""
        import torch.distributed as dist
        if self.reduce not in ("nccl", "multimem"):
            raise ValueError(f"unknown dW reduction {self.reduce!r}")
        seeds = self.seeds(i)
        pending, out = [], []
        mm = self.reduce == "multimem" and self.world > 1
        if mm:
            shapes = [tuple(W.shape) for _, W, _ in data]
            if self.reducer is None or self.reducer.shapes != shapes:
                self.reducer = MulticastReducer(shapes, data[0][1].device, self.group)
            self.reducer.begin()
        for j, (X, W, E) in enumerate(data):
            y, tape = self.linear_fwd(X, W)
            if mm:                            # dW summed over ranks by the wgrad GEMM's epilogue
                view, mc = self.reducer.target(j)
                dx, dw = self.linear_bwd(tape, E, seeds, dw_out=view, dw_accumulate="multimem",
                                         dw_multicast_ptr=mc)
            else:
                dx, dw = self.linear_bwd(tape, E, seeds)
                if self.world > 1:            # the one exchange: dW, overlapping the next projection
                    pending.append(dist.all_reduce(dw, group=self.group, async_op=True))
            out.append((y, dx, dw))
        if mm:
            self.reducer.finish()
        for h in pending:
            h.wait()
        self.last = out
        return out
