"""CPU tests of the product library: it loads without a GPU, exports every
symbol include/mfadd_b200.h declares, fails loudly (no CPU fallback) when no
device exists, and its host-side partition() is bit-exact with the reference
(layout.cpp:217-342) on every BASELINE config and a seeded random sweep
re-expressing test_layout.cpp:141-193."""
import math
import os
import re

import numpy as np
import pytest

import paper_2210_06528_b200 as m
from oracle import orc, ref
from paper_2210_06528_b200 import _lib
from paper_2210_06528_b200 import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "mfadd_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(mfadd_\w+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.EXPORTED)
    assert lib.mfadd_abi_version() == 1


def test_no_cpu_fallback_without_device():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(m.CudaError):
        m.Context(0)


def _ref_or_oracle(grid, blocks, p, nc, ov, clamp=False):
    if ref.available():
        return ref.RefDecomposition(grid, blocks, p, nc, ov, clamp)
    return orc.Decomposition(grid, blocks, p, nc, ov, clamp)


def _assert_same_layout(d, r):
    bd = d.block_dims_array()
    rb = r.blockdims()
    assert np.array_equal(bd, rb)
    for k in range(d.rank):
        assert np.array_equal(d.kvs[k].knots, r.knots(k))  # bitwise
        assert np.array_equal(d._holder_ranges(k), r.holder_ranges(k))
    for b in range(d.nblocks):
        assert d.blocks[b].neighbors == r.neighbors(b)
    assert [list(b.coords) for b in d.blocks] == r.coords().tolist()


@pytest.mark.parametrize("name", list(W.CONFIGS))
def test_partition_bit_exact_on_baseline_configs(name):
    cfg = W.CONFIGS[name]
    d = m.partition(cfg.grid, cfg.bounds, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap)
    r = _ref_or_oracle(cfg.grid, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap)
    _assert_same_layout(d, r)
    if ref.available():
        assert np.array_equal(d.exchange_volume(), r.exchange_volume())
        assert d.compression_ratio() == r.compression_ratio()


def test_partition_sizes_match_survey_table():
    # sum|Q_loc|, sum|P_held|, sum n_s
    expect = {"C1": (10948, 280, 48), "C2": (1254400, 78400, 24576), "C3": (28094464, 3511808, 2386944),
              "C4": (631434960, 21024576, 19764864), "C5": (81577024, 5098564, 1720320)}
    for name, (q, pp, ns) in expect.items():
        cfg = W.CONFIGS[name]
        d = m.partition(cfg.grid, cfg.bounds, cfg.blocks, cfg.degree, cfg.nctrl, cfg.overlap)
        ab = W.algorithmic_bytes(cfg, d, 0)
        assert (ab["q_loc"], ab["p_held"], ab["ns_total"]) == (q, pp, ns), name


def test_partition_random_sweep():
    # test_layout.cpp:141-193 (seed 4242): tilings, symmetry, rejection contract
    rng = np.random.default_rng(4242)
    checked = 0
    for trial in range(60):
        d_ = int(rng.integers(1, 4))
        p = int(rng.integers(1, 6))
        blocks = [int(rng.integers(1, 4 if d_ == 3 else 5)) for _ in range(d_)]
        nctrl = [p + 3 + int(rng.integers(0, 4)) for _ in range(d_)]
        overlap = int(rng.integers(0, 2 * p + 1))
        clamp = bool(rng.integers(0, 4) == 0)
        grid = [blocks[k] * nctrl[k] * 3 for k in range(d_)]
        try:
            r = _ref_or_oracle(grid, blocks, p, nctrl, overlap, clamp)
        except Exception:
            with pytest.raises(m.InvalidArgument):
                m.partition(grid, [(0, 1)] * d_, blocks, p, nctrl, overlap, clamp)
            continue
        d = m.partition(grid, [(0, 1)] * d_, blocks, p, nctrl, overlap, clamp)
        _assert_same_layout(d, r)
        # disjoint exact cover of owned controls per dim
        for k in range(d_):
            nxt = 0
            for c in range(blocks[k]):
                blk = next(b for b in d.blocks if b.coords[k] == c)
                assert blk.dims[k].own_lo == nxt
                nxt = blk.dims[k].own_hi
            assert nxt == d.n_ctrl[k]
        # neighbour symmetry
        for b in d.blocks:
            for j in b.neighbors:
                assert b.id in d.blocks[j].neighbors
        checked += 1
    assert checked > 20


def test_layout_known_answers():
    # test_layout.cpp:32-68
    nb = 8
    d = m.partition([64], [(0, 1)], [2], 3, [nb], 1)
    b0, b1 = d.blocks
    assert (b0.dims[0].own_lo, b0.dims[0].own_hi, b1.dims[0].own_lo, b1.dims[0].own_hi) == (0, nb, nb, 2 * nb)
    assert (b0.dims[0].dof_lo, b0.dims[0].dof_hi, b1.dims[0].dof_lo, b1.dims[0].dof_hi) == (0, nb + 2, nb - 2, 2 * nb)
    assert (b0.dims[0].delta_lo, b0.dims[0].delta_hi, b0.dims[0].overlap_hi) == (0, 1, 1)
    assert b0.neighbors == [1] and b1.neighbors == [0]
    shared = []
    d.shared.for_each_shared(lambda dof, ns: shared.append(ns))
    assert shared == [2] * 4
    # test_layout.cpp:92-111: 2x2 -> one MS cluster of (2(w+delta))^2 dofs, weight 1/4
    for p in (2, 3):
        for ov in (0, 2):
            d = m.partition([40, 40], [(0, 1)] * 2, [2, 2], p, [10, 10], ov)
            band = 2 * (m.delta_width(p) + ov)
            ms = []
            d.shared.for_each_shared(lambda dof, ns: ms.append(dof) if ns > 2 else None)
            assert len(ms) == band * band
            assert all(d.shared.weight(x) == 0.25 for x in ms)
    # test_layout.cpp:123-139: compression ratios
    assert m.partition([200, 200], [(0, 1)] * 2, [5, 5], 3, [20, 20], 0).compression_ratio() == 4.0
    eta = m.partition([704, 540, 550], [(0, 1)] * 3, [8, 8, 8], 3, [35, 35, 35], 0).compression_ratio()
    assert round(eta * 10) / 10 == 9.5
    # test_layout.cpp:240-271: clamped interfaces
    d = m.partition([64], [(0, 1)], [2], 3, [8], 0, True)
    assert d.n_ctrl[0] == 15
    assert int((d.kvs[0].knots == 0.5).sum()) == 3
    shared = []
    d.shared.for_each_shared(lambda dof, ns: shared.append((dof, ns)))
    assert shared == [((7,), 2)]
    # 3x3 centre has eight neighbours
    assert len(m.partition([96, 96], [(0, 1)] * 2, [3, 3], 3, [10, 10], 0).blocks[4].neighbors) == 8
    # delta_width
    assert [m.delta_width(p) for p in (1, 2, 3, 5)] == [0, 1, 1, 2]


def test_partition_rejections():
    # test_layout.cpp:228-238 (messages as in the reference)
    with pytest.raises(m.InvalidArgument, match="overlap too large"):
        m.partition([64], [(0, 1)], [2], 3, [6], 6)
    for args in (([10], [2], 3, [8], 0), ([64], [2], 3, [3], 0), ([64], [0], 3, [8], 0), ([64], [2], 3, [8], -1)):
        with pytest.raises(m.InvalidArgument):
            m.partition(args[0], [(0, 1)], *args[1:])


def test_knot_vectors_bit_exact():
    g = np.load(os.path.join(ROOT, "tests", "golden", "knots_collocation.npz"))
    for i in range(int(g["nkv"][0])):
        p, n, cl, cr = (int(x) for x in g[f"kv{i}_meta"])
        assert np.array_equal(m.make_knot_vector(p, n, 0.0, 1.0, bool(cl), bool(cr)).knots, g[f"kv{i}_knots"])


@pytest.mark.parametrize("n", [2, 3, 4, 8])
def test_shard_box_covers_its_blocks(n):
    """The slab a sharded rank uploads (mfadd_shard_box) is exactly the union of
    its blocks' input rows along axis 0 and contains the rows it decodes."""
    dec = m.partition((4096, 512), [(0, 1), (0, 1)], (16, 4), 5, (32, 32), 5)
    bd = dec.block_dims_array()
    for r in range(n):
        blo, bhi, ilo, ihi = m.shard_range(dec, r, n)
        lo, hi = m.shard_box(dec, r, n)
        assert lo == min(int(bd[b, 0, 12]) for b in range(blo, bhi))
        assert hi == max(int(bd[b, 0, 13]) for b in range(blo, bhi))
        assert lo <= ilo < ihi <= hi


@pytest.mark.parametrize("n", [5, 8, 16])
def test_shard_ranges_finer_than_block_rows(n):
    """More ranks than block rows along axis 0: contiguous block-id ranges
    (runtime.cpp:115-121 deals any block count to any worker count), input rows
    split evenly for the decode, slab = fit rows and decode rows."""
    dec = m.partition((96, 100, 104), [(0, 1)] * 3, (4, 4, 4), 3, (12, 12, 13), 3)
    bd = dec.block_dims_array()
    nxt_b, nxt_i = 0, 0
    for r in range(n):
        blo, bhi, ilo, ihi = m.shard_range(dec, r, n)
        lo, hi = m.shard_box(dec, r, n)
        olo, ohi = m.shard_ctrl_rows(dec, r, n)
        assert (blo, ilo) == (nxt_b, nxt_i) and bhi > blo and ihi > ilo
        nxt_b, nxt_i = bhi, ihi
        assert lo == min(min(int(bd[b, 0, 12]) for b in range(blo, bhi)), ilo)
        assert hi == max(max(int(bd[b, 0, 13]) for b in range(blo, bhi)), ihi)
        assert olo == min(int(bd[b, 0, 10]) for b in range(blo, bhi))
        assert ohi == max(int(bd[b, 0, 11]) for b in range(blo, bhi))
        # every exchange plan is symmetric: what r sends to q is what q receives from r
        for q in range(n):
            if q != r:
                assert np.array_equal(m.shard_exchange(dec, r, n, q, False), m.shard_exchange(dec, q, n, r, True))
    assert (nxt_b, nxt_i) == (64, 96)
    with pytest.raises(ValueError):
        m.shard_range(dec, 0, 65)
