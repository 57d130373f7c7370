"""Pin the CPU oracle against the golden vectors produced by the real
reference (tests/golden/make_golden.py).  No GPU needed."""

import numpy as np
import pytest

import oracle
from oracle import reference_trainers as rt
from conftest import golden_names, load_golden


def rel(got, want):
    return float(np.linalg.norm(np.asarray(got) - np.asarray(want))
                 / max(np.linalg.norm(np.asarray(want)), 1e-30))


@pytest.mark.parametrize("name", golden_names())
def test_selectors_bit_exact(name):
    g = load_golden(name)
    tab = oracle.OracleTable.from_ft(g.ft)
    for k, (ind_sel, gptr, grows, map_sel, mst) in enumerate(oracle.build_selectors(tab)):
        assert np.array_equal(ind_sel, g[f"ind_sel{k}"])
        assert np.array_equal(gptr, g[f"group_indptr{k}"])
        assert np.array_equal(grows, g[f"group_rows{k}"])
        assert np.array_equal(map_sel, g[f"map_sel{k}"])
        assert np.array_equal(mst, g[f"map_sel_t{k}"])


@pytest.mark.parametrize("name", golden_names())
def test_materialize_bit_exact(name):
    g = load_golden(name)
    tab = oracle.OracleTable.from_ft(g.ft)
    assert np.array_equal(oracle.materialize(tab), g["materialized"])


@pytest.mark.parametrize("name", [n for n in golden_names() if n != "clusters"])
def test_operators_match_reference(name):
    g = load_golden(name)
    tab = oracle.OracleTable.from_ft(g.ft)
    assert rel(oracle.lmm(tab, g["op_x"]), g["lmm"]) < 1e-12
    assert rel(oracle.rmm(tab, g["op_w"]), g["rmm"]) < 1e-12
    assert rel(oracle.transpose_lmm(tab, g["op_y"]), g["tlmm"]) < 1e-12
    assert rel(oracle.row_sum(tab), g["row_sum"]) < 1e-12
    assert rel(oracle.col_sum(tab), g["col_sum"]) < 1e-12
    assert np.array_equal(oracle.materialize(oracle.elementwise(tab, "square")),
                          g["sq_materialized"])
    assert rel(oracle.lmm(oracle.elementwise(tab, "abs"), g["op_x"]), g["abs_lmm"]) < 1e-12


EW_CASES = (("scale", 2.5), ("divide", 3.0), ("expm1", None), ("logistic_centered", None))


@pytest.mark.parametrize("name", [n for n in golden_names() if n != "clusters"])
@pytest.mark.parametrize("func,scalar", EW_CASES)
def test_elementwise_maps_match_reference(name, func, scalar):
    """The four maps beyond square / abs (reference sparse.py:298-307)."""
    g = load_golden(name)
    tab = oracle.elementwise(oracle.OracleTable.from_ft(g.ft), func, scalar)
    assert np.array_equal(oracle.materialize(tab), g[f"ew_{func}_materialized"])
    assert rel(oracle.lmm(tab, g["op_x"]), g[f"ew_{func}_lmm"]) < 1e-12


def _trainer_cases():
    out = []
    for name in golden_names():
        g = load_golden(name)
        for model in g.meta.get("trainers", {}):
            out.append((name, model))
    return out


@pytest.mark.parametrize("name,model", _trainer_cases())
def test_trainers_match_reference(name, model):
    g = load_golden(name)
    tab = oracle.OracleTable.from_ft(g.ft)
    m = g.meta["trainers"][model]
    y = {"linreg": g["y_lin"], "logreg": g["y_log"]}.get(model)
    res = rt.train(model, tab, iterations=m["iterations"],
                   learning_rate=m["learning_rate"], k_clusters=m["k_clusters"],
                   rank=m["rank"], seed=m["seed"], y=y)
    want = g[f"{model}_loss"]
    assert np.allclose(res["loss_history"], want, rtol=1e-9, atol=1e-12)
    for pname, val in res["parameters"].items():
        ref = g[f"{model}_{pname}"]
        if pname == "assignments":
            assert np.array_equal(val, ref)
        else:
            assert np.allclose(val, ref, rtol=1e-8, atol=1e-12)


def test_golden_literal_two_source():
    """conftest.py:12-31 golden literal."""
    g = load_golden("two_source")
    want = np.array([[1, 2, 10, 0], [3, 4, 10, 0], [5, 6, 30, 40], [7, 8, 30, 40]], float)
    assert np.array_equal(g["materialized"], want)


def test_kmeans_tie_golden():
    """test_trainers.py:261-270: [[0],[0],[10]], k=3 -> [0,0,2], loss 0."""
    from paper_2502_01985_b200.metadata import FactorizedTable, block_mapping, fk_indicator
    from paper_2502_01985_b200.sparse import SparseMatrix
    s = SparseMatrix.from_dense([[0.0], [0.0], [10.0]])
    ft = FactorizedTable([s], [block_mapping(1, 1, 0)], [fk_indicator(3, 3, [0, 1, 2])],
                         "inner", 3, 1)
    res = rt.kmeans(oracle.OracleTable.from_ft(ft), 3, 3, 0)
    assert np.array_equal(res["parameters"]["assignments"], [0, 0, 2])
    assert res["parameters"]["centroids"][1, 0] == 0.0
    assert res["loss_history"][-1] == 0.0
