"""Multi-GPU: right-hand-side sharding across the GPUs of one box.

One process per GPU (torchrun), ``torch.distributed`` with the NCCL backend
for the only exchange on the path: a broadcast of A from the source rank
(NVLink 5 / NVSwitch).  Right-hand sides are independent (Left: columns of
B, base_kernels.cpp:73-88 and gemm.cpp:185-215; Right: rows of B), so each
rank runs the unchanged single-GPU recursion on its contiguous block and no
reduction follows.  Because every kernel's per-element arithmetic order is
independent of the number of right-hand sides, the P-GPU result is bitwise
identical to the 1-GPU result (the reference's par == seq guarantee,
test_recursion.cpp:421-432, lifted to GPUs).
"""
from __future__ import annotations

from typing import Callable, Optional, Tuple

import torch
import torch.distributed as dist

from .api import Backend, MatrixView, Side, Threshold, TriangularSpec, rec_trmm, rec_trsm


def shard_range(total: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous block [lo, hi) of `total` right-hand sides owned by `rank`
    (sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return total * rank // world, total * (rank + 1) // world


def rhs_count(spec: TriangularSpec, B_rows: int, B_cols: int) -> int:
    return B_cols if Side(spec.side) == Side.Left else B_rows


def broadcast_a(A: torch.Tensor, src: int = 0, group=None) -> None:
    """The single collective: A (its whole storage) from `src` to every rank."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.broadcast(A, src=src, group=group)


def rec_sharded(op: str, spec: TriangularSpec, A: MatrixView, B_local: MatrixView,
                threshold: Threshold = Threshold(), backend: Optional[Backend] = None, src: int = 0,
                group=None, solver: Optional[Callable] = None) -> None:
    """Broadcasts A's origin storage from `src`, then solves/multiplies this
    rank's right-hand-side block in place.  `B_local` holds exactly the block
    ``shard_range(rhs, world, rank)`` of the global B.  `solver` defaults to
    the GPU path (rec_trsm / rec_trmm); it exists so the host logic can be
    exercised by gloo tests on CPU hosts."""
    broadcast_a(A.origin, src=src, group=group)
    fn = solver or (rec_trsm if op == "trsm" else rec_trmm)
    fn(spec, A, B_local, threshold, backend)
