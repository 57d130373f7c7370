"""On-disk / CSV formats against files and results
produced by the REAL reference (tests/golden/formats/, made by
tests/golden/make_formats_golden.py): Matrix Market and ILG1 read exactly and
written byte-identically, a reference-saved dataset directory loads to the
same target, CSV star (inner / left / outer) and union ingestion give the
reference's sources, indicators and materialized targets exactly."""

import json
import os
import shutil

import numpy as np
import pytest

from conftest import GOLDEN_DIR, load_golden
from paper_2502_01985_b200 import formats as fm
from paper_2502_01985_b200.metadata import FactorizedTable

FD = os.path.join(GOLDEN_DIR, "formats")
EXP = np.load(os.path.join(FD, "expected.npz"))


def dense_target(ft: FactorizedTable) -> np.ndarray:
    out = np.zeros((ft.r_T, ft.c_T))
    for s, m, i in zip(ft.sources, ft.mappings, ft.indicators):
        out += i.matrix.to_dense() @ s.to_dense() @ m.matrix.to_dense().T
    return out


@pytest.mark.parametrize("name", ["sparse", "dense", "empty"])
@pytest.mark.parametrize("ext", ["mtx", "ilg"])
def test_matrix_files_read_exact(name, ext):
    a = fm.load_matrix(os.path.join(FD, f"{name}.{ext}"))
    assert [a.n_rows, a.n_cols] == EXP[f"{name}__shape"].tolist()
    for k in ("indptr", "indices", "data"):
        assert np.array_equal(getattr(a, k), EXP[f"{name}__{k}"])


@pytest.mark.parametrize("name", ["sparse", "dense", "empty"])
@pytest.mark.parametrize("ext", ["mtx", "ilg"])
def test_matrix_files_write_byte_identical(name, ext, tmp_path):
    src = os.path.join(FD, f"{name}.{ext}")
    a = fm.load_matrix(src)
    out = tmp_path / f"x.{ext}"
    fm.save_matrix(out, a)
    assert open(out, "rb").read() == open(src, "rb").read()


def test_reference_dataset_directory_loads(tmp_path):
    ft, man = fm.load_dataset(os.path.join(FD, "ds_outer"))
    assert man["format"] == fm.MANIFEST_FORMAT and man["id"] == "ds_outer"
    assert ft.join_type == "outer"
    assert np.array_equal(dense_target(ft), EXP["ds_outer__T"])
    # save -> byte-identical files and manifest, loads back the same
    fm.save_dataset(ft, tmp_path / "copy", dataset_id="ds_outer",
                    generator_params=man.get("generator_params"))
    for f in sorted(os.listdir(os.path.join(FD, "ds_outer"))):
        assert open(tmp_path / "copy" / f, "rb").read() == \
            open(os.path.join(FD, "ds_outer", f), "rb").read(), f
    assert fm.list_datasets(tmp_path) == [str(tmp_path / "copy" / "manifest.json")]


@pytest.mark.parametrize("jt", ["inner", "left", "outer"])
def test_star_csv_ingestion_matches_reference(jt):
    ft = fm.ingest_csv_file(os.path.join(FD, f"star_{jt}.json"))
    assert ft.join_type == jt
    assert np.array_equal(dense_target(ft), EXP[f"star_{jt}__T"])
    for k, (s, i) in enumerate(zip(ft.sources, ft.indicators)):
        assert np.array_equal(s.to_dense(), EXP[f"star_{jt}__src{k}"])
        assert np.array_equal(i.matrix.to_dense(), EXP[f"star_{jt}__ind{k}"])


def test_union_csv_ingestion_matches_reference():
    ft = fm.ingest_csv_file(os.path.join(FD, "union.json"))
    assert ft.join_type == "union"
    assert np.array_equal(dense_target(ft), EXP["union__T"])


def test_csv_errors(tmp_path):
    for f in ("fact.csv", "customers.csv", "products.csv"):
        shutil.copy(os.path.join(FD, f), tmp_path / f)
    m = json.load(open(os.path.join(FD, "star_inner.json")))
    bad = dict(m, join_type="theta")
    with pytest.raises(fm.DatasetError):
        fm.ingest_csv(bad, base_dir=str(tmp_path))
    k = json.loads(json.dumps(m))
    del k["fact"]["keys"]["products"]
    with pytest.raises(fm.DatasetError, match="keys"):
        fm.ingest_csv(k, base_dir=str(tmp_path))
    (tmp_path / "customers.csv").write_text("id,age,income\nc1,25,50\nc1,30,60\n")
    with pytest.raises(fm.DatasetError, match="duplicate"):
        fm.ingest_csv(m, base_dir=str(tmp_path))
    shutil.copy(os.path.join(FD, "customers.csv"), tmp_path / "customers.csv")
    (tmp_path / "fact.csv").write_text("amount,qty,cust,prod\nten,1,c1,p1\n")
    with pytest.raises(fm.DatasetError, match="non-numeric"):
        fm.ingest_csv(m, base_dir=str(tmp_path))
    (tmp_path / "fact.csv").write_text("amount,qty,cust,prod\n1,1,zz,yy\n")
    with pytest.raises(fm.DatasetError, match="no rows"):
        fm.ingest_csv(m, base_dir=str(tmp_path))
    with pytest.raises(fm.DatasetError):
        fm.ingest_csv({"join_type": "union", "tables": []})


def test_matrix_file_errors(tmp_path):
    p = tmp_path / "bad.mtx"
    p.write_text("garbage\n")
    with pytest.raises(fm.FormatError, match="banner"):
        fm.read_matrix_market(p)
    p.write_text("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n")
    with pytest.raises(fm.FormatError, match="declared"):
        fm.read_matrix_market(p)
    q = tmp_path / "bad.ilg"
    q.write_bytes(b"XXXX")
    with pytest.raises(fm.FormatError, match="magic"):
        fm.read_binary(q)


def test_golden_table_roundtrip_through_dataset(tmp_path):
    g = load_golden("gen_union_3_1")
    fm.save_dataset(g.ft, tmp_path / "d", dataset_id="x")
    back, _ = fm.load_dataset(tmp_path / "d")
    assert np.array_equal(dense_target(back), dense_target(g.ft))


@pytest.mark.gpu
def test_ingested_tables_on_device():
    """Datasets loaded from disk / CSV go straight to the B200 path: lmm and
    the materialized join agree with the dense target exactly."""
    import paper_2502_01985_b200 as fl
    for ft in (fm.load_dataset(os.path.join(FD, "ds_outer"))[0],
               fm.ingest_csv_file(os.path.join(FD, "star_outer.json"))):
        h = fl.TargetHandle.factorized(ft)
        T = dense_target(ft)
        assert np.array_equal(fl.as_dense(h.materialize_target()), T.astype(np.float32))
        x = np.arange(ft.c_T * 2, dtype=np.float64).reshape(ft.c_T, 2) / 7.0
        got = fl.as_dense(h.lmm(x))
        assert np.allclose(got, T @ x, rtol=1e-5, atol=1e-5)
