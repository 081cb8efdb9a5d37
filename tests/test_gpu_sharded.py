"""Sharded (multi-GPU) solve, all ranks in one process on one device with the
loopback transport (device copies in place of NCCL, host-ordered steps): the
per-epoch cross-rank exchange and the dp max-reduction must reproduce the
single-device solve."""
import numpy as np
import pytest

import paper_2210_06528_b200 as m
from paper_2210_06528_b200 import workloads as W

pytestmark = pytest.mark.gpu

CASES = [
    # rank counts above the block rows along axis 0 (4 for C2s / C3s) cut block
    # rows: contiguous block-id ranges, holders on any neighbouring rank
    ("C2s", W.scaled(W.CONFIGS["C2"], (400, 380), (20, 18)), (2, 4, 5, 8, 16)),
    ("C3s", W.scaled(W.CONFIGS["C3"], (96, 100, 104), (12, 12, 13)), (2, 3, 5, 8)),
    ("C5s", W.scaled(W.CONFIGS["C5"], (1536, 1408), (24, 22)), (2, 3, 8)),
]


@pytest.mark.parametrize("name,cfg,ranks", CASES, ids=[c[0] for c in CASES])
def test_loopback_matches_single_device(ctx, name, cfg, ranks):
    values = W.make_field_numpy(cfg)
    dec = m.partition(cfg.grid, cfg.bounds, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap)
    scfg = m.SolverConfig(max_outer_iterations=cfg.max_iters, tolerance=cfg.tolerance, log_errors=False)
    f = m.Field(list(cfg.grid), list(cfg.bounds), values)
    ref = m.solve(f, dec, scfg)
    for n in ranks:
        r = m.solve_loopback(f, dec, n, scfg)
        # identical ordered sums on both ranks of every cross-rank region
        assert np.array_equal(r.model.controls, ref.model.controls), (name, n)
        assert r.converged == ref.converged and r.constraint_iterations == ref.constraint_iterations
        assert [e.dp_max for e in r.epochs] == [e.dp_max for e in ref.epochs]
        assert [(e.jump_ss, e.jump_ms) for e in r.epochs] == [(e.jump_ss, e.jump_ms) for e in ref.epochs]
        assert [(j.block_a, j.block_b, j.linf_ss, j.linf_ms) for j in r.final_jumps] == \
               [(j.block_a, j.block_b, j.linf_ss, j.linf_ms) for j in ref.final_jumps]
        assert np.array_equal(r.global_error, ref.global_error)
        # L2: per-rank partial sums combined in rank order
        assert abs(r.global_l2 - ref.global_l2) <= 1e-12 * ref.global_l2
        assert r.global_linf == ref.global_linf


@pytest.mark.parametrize("max_iters", [1, 2, 4])
def test_loopback_iteration_budget(ctx, max_iters, monkeypatch):
    """The chunked epoch loop (iterations enqueued ahead of the host's read of
    the loop state, predicated on convergence) stops where the single-device
    loop stops: out of budget before convergence, or converged inside a chunk
    (solver.cpp:394-413)."""
    cfg = W.scaled(W.CONFIGS["C2"], (400, 380), (20, 18))
    values = W.make_field_numpy(cfg)
    dec = m.partition(cfg.grid, cfg.bounds, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap)
    f = m.Field(list(cfg.grid), list(cfg.bounds), values)
    scfg = m.SolverConfig(max_outer_iterations=max_iters, tolerance=cfg.tolerance, log_errors=False)
    ref = m.solve(f, dec, scfg)
    for chunk in ("1", "3"):
        monkeypatch.setenv("MFADD_SHARD_CHUNK", chunk)
        for n in (2, 8):
            r = m.solve_loopback(f, dec, n, scfg)
            assert (r.converged, r.constraint_iterations, len(r.epochs)) == \
                   (ref.converged, ref.constraint_iterations, len(ref.epochs)), (max_iters, chunk, n)
            assert [e.dp_max for e in r.epochs] == [e.dp_max for e in ref.epochs]
            assert np.array_equal(r.model.controls, ref.model.controls)
            assert [(j.linf_ss, j.linf_ms) for j in r.final_jumps] == [(j.linf_ss, j.linf_ms) for j in ref.final_jumps]


def test_loopback_enforce_off_and_1d(ctx):
    # decoupled fits (no exchange epochs) still need the final cross-rank jumps
    cfg = W.scaled(W.CONFIGS["C2"], (400, 380), (20, 18))
    values = W.make_field_numpy(cfg)
    dec = m.partition(cfg.grid, cfg.bounds, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap)
    f = m.Field(list(cfg.grid), list(cfg.bounds), values)
    scfg = m.SolverConfig(max_outer_iterations=20, log_errors=False, enforce_continuity=False)
    ref = m.solve(f, dec, scfg)
    r = m.solve_loopback(f, dec, 2, scfg)
    assert np.array_equal(r.model.controls, ref.model.controls)
    assert [(j.linf_ss, j.linf_ms) for j in r.final_jumps] == [(j.linf_ss, j.linf_ms) for j in ref.final_jumps]
    # 1-D, converges after one constraint iteration: final jumps from the exchange
    cfg1 = W.CONFIGS["C1"]
    v1 = W.make_field_numpy(cfg1)
    dec1 = m.partition(cfg1.grid, cfg1.bounds, cfg1.blocks, cfg1.degree, cfg1.nctrl, cfg1.overlap)
    f1 = m.Field(list(cfg1.grid), list(cfg1.bounds), v1)
    s1 = m.SolverConfig(max_outer_iterations=20, log_errors=False)
    ref1 = m.solve(f1, dec1, s1)
    for n in (2, 4):
        r1 = m.solve_loopback(f1, dec1, n, s1)
        assert np.array_equal(r1.model.controls, ref1.model.controls)
        assert [(j.linf_ss, j.linf_ms) for j in r1.final_jumps] == [(j.linf_ss, j.linf_ms) for j in ref1.final_jumps]


def test_nccl_comm_single_rank(ctx):
    """NCCL initialisation and the sharded constructor through the C ABI; with
    one rank the solve must equal the plain solver."""
    cfg = W.scaled(W.CONFIGS["C2"], (400, 380), (20, 18))
    values = W.make_field_numpy(cfg)
    dec = m.partition(cfg.grid, cfg.bounds, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap)
    scfg = m.SolverConfig(max_outer_iterations=20, log_errors=False)
    comm = m.Comm(m.Comm.unique_id(), 0, 1, ctx)
    try:
        s = m.Solver(dec, scfg, ctx, comm=comm)
        s.run(values.reshape(-1))
        r = s.result()
        ref = m.solve(m.Field(list(cfg.grid), list(cfg.bounds), values), dec, scfg)
        assert np.array_equal(r.model.controls, ref.model.controls)
        s.close()
    finally:
        comm.close()
