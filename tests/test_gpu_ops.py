"""GPU parity: the B200 operators vs the reference's golden vectors and the
CPU oracle.  Integer / index work and the join are compared bit-exactly;
floating point at the north-star tolerance (fp32 storage, fp64 reductions)."""

import numpy as np
import pytest

import oracle
from conftest import golden_names, load_golden, star_table

pytestmark = pytest.mark.gpu

RTOL = 1e-5   # operator outputs: fp32 values, fp64 reductions


def rel(got, want):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    return float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30))


@pytest.fixture(scope="module")
def fl():
    import paper_2502_01985_b200 as fl
    return fl


@pytest.mark.parametrize("name", golden_names())
def test_materialize_bit_exact(fl, name):
    g = load_golden(name)
    h = fl.TargetHandle.factorized(g.ft)
    got = h.materialize_dense()
    assert got.dtype == np.float32
    assert np.array_equal(got.astype(np.float64), g["materialized"])


@pytest.mark.parametrize("name", golden_names())
def test_selectors_bit_exact(fl, name):
    """Device-derived selectors (perm, stable sort, scan) == the reference's
    `_build_selectors` output (ops.py:55-74)."""
    g = load_golden(name)
    h = fl.TargetHandle.factorized(g.ft)
    sels = h.selectors
    for k, s in enumerate(sels):
        assert np.array_equal(s.ind_sel, g[f"ind_sel{k}"])
        assert np.array_equal(s.group_indptr, g[f"group_indptr{k}"])
        assert np.array_equal(s.group_rows, g[f"group_rows{k}"])
        assert np.array_equal(s.map_sel, g[f"map_sel{k}"])
        assert np.array_equal(s.map_sel_t, g[f"map_sel_t{k}"])


@pytest.mark.parametrize("name", [n for n in golden_names() if n != "clusters"])
def test_operators_match_reference(fl, name):
    g = load_golden(name)
    h = fl.TargetHandle.factorized(g.ft)
    x = fl.SparseMatrix.from_dense(g["op_x"])
    w = fl.SparseMatrix.from_dense(g["op_w"])
    y = fl.SparseMatrix.from_dense(g["op_y"])
    assert rel(h.lmm(x).to_dense(), g["lmm"]) < RTOL
    assert rel(h.rmm(w).to_dense(), g["rmm"]) < RTOL
    assert rel(h.transpose_lmm(y).to_dense(), g["tlmm"]) < RTOL
    assert rel(h.row_sum().to_dense(), g["row_sum"]) < RTOL
    assert rel(h.col_sum().to_dense(), g["col_sum"]) < RTOL
    sq = h.elementwise("square").materialize_target().to_dense()
    assert rel(sq, g["sq_materialized"]) < 1e-7
    assert rel(h.elementwise("abs").lmm(x).to_dense(), g["abs_lmm"]) < RTOL


EW_CASES = (("scale", 2.5), ("divide", 3.0), ("expm1", None), ("logistic_centered", None),
            ("square", None), ("abs", None))


@pytest.mark.parametrize("name", [n for n in golden_names() if n != "clusters"])
@pytest.mark.parametrize("func,scalar", EW_CASES)
def test_elementwise_maps_match_reference(fl, name, func, scalar):
    """Every registered map (reference sparse.py:298-307) applied on the
    device: the mapped join equals the reference's fp64 map rounded to fp32
    (the device evaluates f in fp64 and stores fp32: relative 2^-24 per
    value), and one product over the mapped table matches at RTOL."""
    g = load_golden(name)
    h = fl.TargetHandle.factorized(g.ft)
    m = h.elementwise(func, scalar)
    got = m.materialize_dense().astype(np.float64)
    if func == "abs":
        assert np.array_equal(got, np.abs(g["materialized"]))      # exact in fp32
        return
    want = g["sq_materialized"] if func == "square" else g[f"ew_{func}_materialized"]
    assert np.array_equal(got == 0, want == 0)          # f(0) = 0: structure kept
    assert np.all(np.abs(got - want) <= 2.0 ** -24 * (1 + 1e-6) * np.abs(want))
    if func != "square":
        assert rel(m.lmm(g["op_x"]), g[f"ew_{func}_lmm"]) < RTOL


def test_spec_examples(fl):
    """test_factorized_ops.py:87-138: lmm(I)=T, rmm(I)=T, rmm(e_i)=row i,
    lmm(1)=rowSum, rmm(1)=colSum, tlmm(I)=T^T."""
    g = load_golden("two_source")
    ref = g["materialized"]
    h = fl.TargetHandle.factorized(g.ft)
    eye = fl.SparseMatrix.identity(4)
    assert np.array_equal(h.lmm(eye).to_dense(), ref)
    assert np.array_equal(h.rmm(eye).to_dense(), ref)
    assert np.array_equal(h.transpose_lmm(eye).to_dense(), ref.T)
    for i in range(4):
        e = fl.SparseMatrix.from_coo(1, 4, [0], [i], [1.0])
        assert np.array_equal(h.rmm(e).to_dense(), ref[i:i + 1])
    ones = fl.SparseMatrix.from_dense(np.ones((4, 1)))
    assert np.allclose(h.lmm(ones).to_dense(), h.row_sum().to_dense())
    ones_r = fl.SparseMatrix.from_dense(np.ones((1, 4)))
    assert np.allclose(h.rmm(ones_r).to_dense(), h.col_sum().to_dense())


def test_outer_padding_row_is_zero(fl):
    g = load_golden("outer")
    h = fl.TargetHandle.factorized(g.ft)
    rs = h.row_sum().to_dense()
    assert rs[4, 0] == 0.0


def test_materialized_handle_matches(fl):
    g = load_golden("star3")
    tmat = fl.SparseMatrix.from_dense(g["materialized"])
    mh = fl.TargetHandle.materialized(tmat)
    assert mh.path == "materialized"
    x = g["op_x"]
    assert rel(mh.lmm(x), g["lmm"]) < RTOL
    assert rel(mh.transpose_lmm(g["op_y"]), g["tlmm"]) < RTOL
    assert rel(mh.rmm(g["op_w"]), g["rmm"]) < RTOL


@pytest.mark.parametrize("name", golden_names())
def test_crossprod_matches_dense(fl, name):
    """Factorized T^T T (no materialization: F^T F, S_d^T diag(n_d) S_d and
    S_d^T (I_d^T [F | I_e S_e]) blocks) against the dense product of the
    reference's materialized join, for every golden table (inner / left /
    outer joins, unions, 2-3 sources)."""
    g = load_golden(name)
    h = fl.TargetHandle.factorized(g.ft)
    td = g["materialized"]
    got = h.crossprod()
    assert got.shape == (td.shape[1], td.shape[1])
    assert rel(got, td.T @ td) < RTOL
    assert np.allclose(got, got.T, rtol=1e-6, atol=0)


@pytest.mark.parametrize("dims,c_fact", [([(1000, 50)], 20), ([(300, 9), (40, 5)], 7),
                                         ([(997, 37), (13, 3)], 29), ([], 45),
                                         ([(50 + i, 2 + i) for i in range(10)], 6)])
def test_crossprod_random_star_vs_oracle(fl, dims, c_fact):
    """Wide tables (several 32-column output tiles), more gathered sources
    than one grouped pass takes (10 > 8), and a fact-only table."""
    ft = star_table(17, 50_003, dims, c_fact)
    tab = oracle.OracleTable.from_ft(ft)
    td = oracle.materialize(tab)
    h = fl.TargetHandle.factorized(ft)
    got = h.crossprod()
    assert rel(got, td.T @ td) < RTOL


def test_shape_errors(fl):
    g = load_golden("two_source")
    h = fl.TargetHandle.factorized(g.ft)
    with pytest.raises(fl.ShapeError):
        h.lmm(np.ones((5, 2)))
    with pytest.raises(fl.ShapeError):
        h.rmm(np.ones((2, 5)))
    with pytest.raises(fl.ShapeError):
        h.transpose_lmm(np.ones((3, 2)))
    with pytest.raises(fl.OpError, match="materialization"):
        h.elementwise("logistic")


def test_invalid_metadata_rejected(fl):
    from paper_2502_01985_b200.metadata import MetadataError
    s1 = fl.SparseMatrix.from_dense([[1.0, 2.0]])
    s2 = fl.SparseMatrix.from_dense([[3.0, 4.0]])
    m1 = fl.MappingMatrix(fl.SparseMatrix.from_dense([[1, 0], [0, 1], [0, 0]]))
    m2 = fl.MappingMatrix(fl.SparseMatrix.from_dense([[0, 0], [1, 0], [0, 1]]))
    i = fl.IndicatorMatrix(fl.SparseMatrix.from_dense([[1.0]]))
    bad = fl.FactorizedTable([s1, s2], [m1, m2], [i, i], "inner", 1, 3)
    with pytest.raises(MetadataError):
        fl.TargetHandle.factorized(bad)


@pytest.mark.parametrize("dims,sort_fk", [([(1000, 13)], False), ([(700, 9), (60, 5)], False),
                                          ([(50, 7)], True), ([(3, 4), (997, 6)], False)])
def test_random_star_vs_oracle(fl, dims, sort_fk):
    """Larger random star schemas (several tiles and CTAs, segments crossing
    tiles and CTAs) vs the oracle."""
    ft = star_table(5, 150_000, dims, 21, sort_fk=sort_fk)
    tab = oracle.OracleTable.from_ft(ft)
    h = fl.TargetHandle.factorized(ft)
    rng = np.random.default_rng(0)
    x = rng.random((ft.c_T, 3)).astype(np.float32)
    y = rng.random((ft.r_T, 2)).astype(np.float32)
    w = rng.random((2, ft.r_T)).astype(np.float32)
    assert rel(h.lmm(x), oracle.lmm(tab, x)) < RTOL
    assert rel(h.transpose_lmm(y), oracle.transpose_lmm(tab, y)) < RTOL
    assert rel(h.rmm(w), oracle.rmm(tab, w)) < RTOL
    assert np.array_equal(h.materialize_dense().astype(np.float64), oracle.materialize(tab))


@pytest.mark.parametrize("chunk", [None, "4096", "80"])
def test_upload_paths_agree(fl, monkeypatch, chunk):
    """The same table uploaded from pageable numpy, pinned host tensors and
    device tensors joins to the identical T (bit-exact).  Host values travel
    in ring chunks (FL_UPLOAD_CHUNK_BYTES forces many ring wraps and one-row
    chunks); the fact source is injective but NOT the identity (outer-join
    padding rows, shuffled), so the scatter goes through the inverted
    indicator."""
    import torch
    if chunk is not None:
        monkeypatch.setenv("FL_UPLOAD_CHUNK_BYTES", chunk)
    rng = np.random.default_rng(7)
    r_fact, c_fact, r_dim, c_dim, r_extra = 3001, 7, 97, 5, 40
    r_t, c_t = r_fact + r_extra, c_fact + c_dim
    fact = rng.random((r_fact, c_fact)).astype(np.float32)
    dim = rng.random((r_dim, c_dim)).astype(np.float32)
    sel_f = np.full(r_t, -1, np.int32)
    sel_f[rng.permutation(r_t)[:r_fact]] = np.arange(r_fact, dtype=np.int32)
    sel_d = rng.integers(-1, r_dim, r_t).astype(np.int32)
    maps = [np.arange(c_fact, dtype=np.int32), np.arange(c_fact, c_t, dtype=np.int32)]
    want = np.zeros((r_t, c_t), np.float32)
    m = sel_f >= 0
    want[m, :c_fact] = fact[sel_f[m]]
    m = sel_d >= 0
    want[m, c_fact:] = dim[sel_d[m]]
    pinned = lambda a: torch.from_numpy(a).pin_memory()  # noqa: E731
    variants = {
        "numpy": ([fact, dim], [sel_f, sel_d]),
        "pinned": ([pinned(fact), pinned(dim)], [pinned(sel_f), pinned(sel_d)]),
        "cuda": ([torch.from_numpy(fact).cuda(), torch.from_numpy(dim).cuda()],
                 [torch.from_numpy(sel_f).cuda(), torch.from_numpy(sel_d).cuda()]),
    }
    for name, (srcs, sels) in variants.items():
        srcs = [s.numpy() if hasattr(s, "is_pinned") and not s.is_cuda else s for s in srcs]
        sels = [s.numpy() if hasattr(s, "is_pinned") and not s.is_cuda else s for s in sels]
        h = fl.TargetHandle.from_arrays(srcs, sels, maps, r_t, c_t)
        got = h.materialize_dense()
        assert np.array_equal(got, want), name
        # identity fact indicator as well (the star-schema fast path)
        h2 = fl.TargetHandle.from_arrays([srcs[0], srcs[1]], [None, sels[1][:r_fact]], maps,
                                         r_fact, c_t)
        w2 = np.zeros((r_fact, c_t), np.float32)
        w2[:, :c_fact] = fact
        m2 = sel_d[:r_fact] >= 0
        w2[m2, c_fact:] = dim[sel_d[:r_fact][m2]]
        assert np.array_equal(h2.materialize_dense(), w2), name + " identity"


@pytest.mark.parametrize("c_fact,dims", [(20, [(1000, 50)]), (7, [(300, 9), (40, 5)]),
                                         (29, [(997, 6)]), (3, [])])
def test_narrow_lmm_matches_generic(fl, monkeypatch, c_fact, dims):
    """The thread-per-row lmm (device-order output + gathered unpermute,
    forced on here via FL_LMM_NARROW_MIN_ROWS=0) is bit-identical to the
    generic kernel and matches the oracle, for 1-9, 15, 16, 20, 32 and 33
    operand columns (1-4: thread-per-row kernel; 16-32 per chunk: the
    warp-per-row kernel; 5-15 the generic kernel)."""
    ft = star_table(11, 70_001, dims, c_fact)
    tab = oracle.OracleTable.from_ft(ft)
    h = fl.TargetHandle.factorized(ft)
    rng = np.random.default_rng(1)
    monkeypatch.setenv("FL_LMM_NARROW_MIN_ROWS", "0")
    for cx in (1, 2, 3, 4, 5, 6, 7, 8, 9, 15, 16, 20, 32, 33):
        x = rng.random((ft.c_T, cx)).astype(np.float32)
        got = h.lmm(x)
        monkeypatch.setenv("FL_NO_NARROW_LMM", "1")
        generic = h.lmm(x)
        monkeypatch.delenv("FL_NO_NARROW_LMM")
        assert np.array_equal(got, generic), cx
        assert rel(got, oracle.lmm(tab, x)) < RTOL


@pytest.mark.parametrize("c_fact", [20, 8, 32, 13])
def test_transpose_lmm_widths_vs_oracle(fl, c_fact):
    """T^T y for 1-9 y columns: the stream block takes the thread-per-row
    kernel one column pair per pass (up to 8 columns, stream pitch <= 32),
    wider y or stream blocks the staged generic kernel."""
    ft = star_table(12, 60_003, [(900, 11), (31, 4)], c_fact)
    tab = oracle.OracleTable.from_ft(ft)
    h = fl.TargetHandle.factorized(ft)
    rng = np.random.default_rng(2)
    for cy in range(1, 10):
        y = rng.random((ft.r_T, cy)).astype(np.float32)
        assert rel(h.transpose_lmm(y), oracle.transpose_lmm(tab, y)) < RTOL, cy


@pytest.mark.parametrize("c_fact,dims", [(20, [(2000, 30)]), (12, [(500, 7), (40, 3)]),
                                         (28, []), (5, [(3000, 9)])])
def test_lmm_tcgen05_vs_oracle(fl, monkeypatch, c_fact, dims):
    """The tcgen05 lmm (csrc/lmm_t5.cuh: F x_F as a 3xTF32 tcgen05 MMA per
    128-row tile, gathered q_d rows added in the epilogue, rows written at
    their target positions), forced on here (FL_LMM_T5=1, FL_LMM_T5_MIN_ROWS=0), for
    8-40 operand columns (chunks of 32, ragged last chunk, odd widths)."""
    monkeypatch.setenv("FL_LMM_T5", "1")
    monkeypatch.setenv("FL_LMM_T5_MIN_ROWS", "0")
    ft = star_table(13, 50_001, dims, c_fact)
    tab = oracle.OracleTable.from_ft(ft)
    h = fl.TargetHandle.factorized(ft)
    rng = np.random.default_rng(2)
    for cx in (8, 13, 16, 32, 33, 40):
        x = rng.random((ft.c_T, cx)).astype(np.float32)
        got = h.lmm(x)
        assert rel(got, oracle.lmm(tab, x)) < RTOL, cx
        monkeypatch.setenv("FL_LMM_T5", "2")   # device-order rows + row gather: same values
        assert np.array_equal(h.lmm(x), got), cx
        monkeypatch.setenv("FL_LMM_T5", "1")


@pytest.mark.parametrize("c_fact,dims", [(20, [(2000, 30)]), (28, []), (3, [(500, 7), (40, 3)])])
def test_crossprod_tcgen05_gram_matches_simt(fl, monkeypatch, c_fact, dims):
    """F^T F of the crossprod on tcgen05 (csrc/gram_t5.cuh: [F | F_lo]^T
    [F | F_lo] read MN-major per 128-row tile) against the SIMT tile Gram
    (FL_NO_GRAM_T5=1) and the dense product."""
    ft = star_table(19, 90_001, dims, c_fact)
    tab = oracle.OracleTable.from_ft(ft)
    td = oracle.materialize(tab)
    h = fl.TargetHandle.factorized(ft)
    got = h.crossprod()
    monkeypatch.setenv("FL_GRAM_TMA", "1")   # 2-D TMA tiles instead of bulk-copied rows
    monkeypatch.setenv("FL_GRAM_M64", "1")   # M = 64 MMA shape (16-lane TMEM quadrants)
    got64 = h.crossprod()
    monkeypatch.delenv("FL_GRAM_M64")
    got_tma = h.crossprod()
    monkeypatch.delenv("FL_GRAM_TMA")
    assert rel(got, got_tma) < 4e-6
    monkeypatch.setenv("FL_NO_GRAM_T5", "1")
    simt = h.crossprod()
    assert rel(got, td.T @ td) < RTOL
    assert rel(got, simt) < 4e-6
    assert rel(got64, simt) < 4e-6


@pytest.mark.parametrize("c_fact,dims,sort_fk", [(20, [(2000, 30)], False), (28, [], False),
                                                 (13, [(500, 7), (40, 3)], False),
                                                 (3, [(3000, 9)], True)])
def test_wide_tlmm_rmm_tcgen05_vs_oracle(fl, monkeypatch, c_fact, dims, sort_fk):
    """Wide T^T y and rmm through the tcgen05 pass (csrc/tmm_t5.cuh: y laid
    out once in device order, [F | F_lo | Y | Y_lo]^T [Y | Y_lo] per 128-row
    tile) for 3..32 operand columns, against the oracle and against the
    per-column-pair SIMT passes (FL_NO_TMM_T5=1); 33 columns stays on the
    chunked path."""
    ft = star_table(23, 70_001, dims, c_fact, sort_fk=sort_fk)
    tab = oracle.OracleTable.from_ft(ft)
    h = fl.TargetHandle.factorized(ft)
    rng = np.random.default_rng(4)
    for cy in (3, 5, 9, 16, 31, 32, 33):
        y = rng.random((ft.r_T, cy)).astype(np.float32)
        w = rng.random((cy, ft.r_T)).astype(np.float32)
        got_t = h.transpose_lmm(y)
        got_r = h.rmm(w)
        assert rel(got_t, oracle.transpose_lmm(tab, y)) < RTOL, cy
        assert rel(got_r, oracle.rmm(tab, w)) < RTOL, cy
        monkeypatch.setenv("FL_NO_TMM_T5", "1")
        assert rel(got_t, h.transpose_lmm(y)) < 4e-6, cy
        assert rel(got_r, h.rmm(w)) < 4e-6, cy
        monkeypatch.delenv("FL_NO_TMM_T5")
