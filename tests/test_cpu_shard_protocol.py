"""Multi-rank exchange protocol of the sharded solve, on CPU with gloo.

Two (or three) processes each own a slab of block rows (mfadd_shard_range) and
run the epoch loop of solver.cpp:394-413 in numpy on their blocks' decoupled
fits, exchanging the copies of cross-rank shared controls in exactly the
buffer layout the GPU path packs (mfadd_shard_exchange: the same
mfb::shard_peers plan), with dp max-reduced over ranks.  The result must equal
the single-process reference enforcement (oracle) bitwise: every rank forms
the same ascending-holder sum for a shared control.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2210_06528_b200 as m
from oracle import orc

CASES = {
    "2d": ([160, 150], [4, 3], 3, [10, 12], 2),
    "3d": ([40, 36, 30], [3, 2, 2], 2, [7, 6, 6], 1),
}


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _field(grid):
    return np.random.default_rng(20221012).standard_normal(grid)


def _local_index(dec, b, gidx):
    return tuple(int(g) - dec.blocks[b].dims[k].dof_lo for k, g in enumerate(gidx))


def _worker(rank, nranks, port, case, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=nranks)
    try:
        import torch
        grid, blocks, p, nc, ov = CASES[case]
        D = len(grid)
        dec = m.partition(grid, [(0, 1)] * D, blocks, p, nc, ov)
        od = orc.Decomposition(grid, blocks, p, nc, ov)
        values = _field(grid)
        fits = orc.solve(od, values, 20, 1e-10, enforce_continuity=False).blocks_p  # decoupled local fits
        ref = orc.solve(od, values, 20, 1e-10)
        blo, bhi, _, _ = m.shard_range(dec, rank, nranks)
        P = {b: fits[b].copy() for b in range(blo, bhi)}
        peers = [q for q in range(nranks) if q != rank]
        plans = {q: (m.shard_exchange(dec, rank, nranks, q, False), m.shard_exchange(dec, rank, nranks, q, True))
                 for q in peers}
        # shared controls held by a local block, each with its ascending holders
        shared = {}
        for b in range(blo, bhi):
            lo = [d.dof_lo for d in dec.blocks[b].dims]
            for li in np.ndindex(P[b].shape):
                g = tuple(lo[k] + li[k] for k in range(D))
                if g not in shared and dec.shared.n_s(g) >= 2:
                    shared[g] = dec.shared.holders(g)

        def exchange():
            remote = {}
            for q in peers:
                send, recv = plans[q]
                buf = np.array([P[int(e[0])][_local_index(dec, int(e[0]), e[1:1 + D])] for e in send], np.float64)
                rbuf = np.zeros(len(recv), np.float64)
                ts, tr = torch.from_numpy(buf), torch.from_numpy(rbuf)
                reqs = []
                if len(buf):
                    reqs.append(dist.isend(ts, q))
                if len(rbuf):
                    reqs.append(dist.irecv(tr, q))
                for r_ in reqs:
                    r_.wait()
                for e, v in zip(recv, tr.numpy()):
                    remote[(int(e[0]), tuple(int(x) for x in e[1:1 + D]))] = float(v)
            return remote

        iters, converged, dps = 0, False, []
        for it in range(1, 21):
            remote = exchange()  # Jacobi snapshot: every copy as of the previous epoch
            change = {b: 0.0 for b in P}
            updates = []
            for g, hold in shared.items():
                ns = len(hold)
                if it == 1 and ns != 2:  # solver.cpp:397: first iteration averages n_s == 2 only
                    continue
                vals = [P[h][_local_index(dec, h, g)] if h in P else remote[(h, g)] for h in hold]
                s = 0.0
                for v in vals:  # ascending holder id, divide once (solver.cpp:147-159)
                    s = s + v
                avg = s / ns
                for h, v in zip(hold, vals):
                    if h in P:
                        change[h] = max(change[h], abs(avg - v))
                        updates.append((h, _local_index(dec, h, g), avg))
            for h, li, avg in updates:
                P[h][li] = avg
            dp = max([change[b] / max(1.0, float(np.abs(P[b]).max())) for b in P] + [0.0])
            t = torch.tensor([dp], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dps.append(float(t.item()))
            iters = it
            if dps[-1] < 1e-10:
                converged = True
                break
        ok = all(np.array_equal(P[b], ref.blocks_p[b]) for b in P)
        ref_dps = [float(e[1]) for e in np.asarray(ref.epochs)[1:]]  # rows (iteration, dp, jump_ss, jump_ms)
        out[rank] = (ok, converged == bool(ref.converged), iters - 1 if converged else iters,
                     ref.constraint_iterations, np.allclose(dps, ref_dps, rtol=0, atol=0))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case,nranks", [("2d", 2), ("2d", 3), ("3d", 2), ("2d", 5)])
def test_gloo_shard_protocol_matches_reference(case, nranks):
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    port = _free_port()
    mp.start_processes(_worker, args=(nranks, port, case, out), nprocs=nranks, join=True, start_method="spawn")
    assert len(out) == nranks
    for r in range(nranks):
        ok, conv_eq, iters, ref_iters, dps_eq = out[r]
        assert ok, f"rank {r}: blocks differ from the single-process enforcement"
        assert conv_eq and iters == ref_iters and dps_eq
