"""Multi-process (world size 2, gloo, CPU) test of the RHS-sharding host
logic in paper_2504_13821_b200/dist.py: shard ranges, the broadcast of A and
per-rank solves reassemble bitwise into the unsharded result.  The per-rank
compute here is the ORACLE (test-only stand-in, no GPU on CPU hosts); on the
GPU box the same function runs the sm_100a path."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2504_13821_b200 import MatrixBuffer, Side, Threshold, TriangularSpec, Uplo
from paper_2504_13821_b200.dist import rec_sharded, rhs_count, shard_range


def test_shard_range_partitions():
    for total in (0, 1, 7, 16384, 524288):
        for world in (1, 2, 4, 8):
            spans = [shard_range(total, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == total
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


def _oracle_solver(op):
    def solve(spec, A, B, threshold, backend):
        a = np.asfortranarray(A.tensor().numpy())
        b = np.asfortranarray(B.tensor().numpy())
        s = oracle.spec(int(spec.side), int(spec.uplo), int(spec.trans), int(spec.diag), spec.alpha)
        out = oracle.oracle_trsm(s, a, b) if op == "trsm" else oracle.oracle_trmm(s, a, b)
        B.tensor().copy_(torch.from_numpy(out))
    return solve


def _worker(rank, world, port, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, m = 24, 10
        for op, side in (("trsm", Side.Left), ("trmm", Side.Right)):
            spec = TriangularSpec(side, Uplo.Lower, alpha=1.25)
            # rank 0 owns A; others start with zeros and receive it.
            a = oracle.make_dominant(n, 0, 5) if rank == 0 else np.zeros((n, n), order="F")
            A = MatrixBuffer.from_tensor(torch.from_numpy(np.ascontiguousarray(a)), device="cpu")
            full = oracle.make_random(n, m, 6) if side == Side.Left else oracle.make_random(m, n, 6)
            total = rhs_count(spec, *full.shape)
            lo, hi = shard_range(total, world, rank)
            local = full[:, lo:hi] if side == Side.Left else full[lo:hi, :]
            B = MatrixBuffer.from_tensor(torch.from_numpy(np.ascontiguousarray(local)), device="cpu")
            rec_sharded(op, spec, A.cview(), B.view(), Threshold(4), solver=_oracle_solver(op))
            results[f"{op}-{rank}"] = (lo, hi, B.numpy().copy(), A.numpy().copy())
    finally:
        dist.destroy_process_group()


def test_two_rank_sharding_matches_unsharded():
    world = 2
    port = 29500 + os.getpid() % 1000
    with mp.Manager() as mgr:
        results = mgr.dict()
        mp.spawn(_worker, args=(world, port, results), nprocs=world, join=True)
        results = dict(results)
    n, m = 24, 10
    a = oracle.make_dominant(n, 0, 5)
    for op, side in (("trsm", 0), ("trmm", 1)):
        s = oracle.spec(side, 0, 0, 0, 1.25)
        full = oracle.make_random(n, m, 6) if side == 0 else oracle.make_random(m, n, 6)
        want = oracle.oracle_trsm(s, a, full) if op == "trsm" else oracle.oracle_trmm(s, a, full)
        parts = []
        for r in range(world):
            lo, hi, blk, a_seen = results[f"{op}-{r}"]
            assert np.array_equal(a_seen, a)  # the broadcast delivered A
            parts.append(blk)
        got = np.concatenate(parts, axis=1 if side == 0 else 0)
        assert np.array_equal(got, want)
