"""Golden fixtures for the on-disk / CSV formats, made
by the REAL reference in the build container:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_formats_golden.py

Writes tests/golden/formats/: Matrix Market and ILG1 files written by the
reference's io.py, a dataset directory saved by its datasets.save_dataset
(a datagen table), star / union CSV inputs, and expected.npz holding the
reference's parse / ingestion results (CSR arrays, dense materialized
targets) for the product's tests to compare against exactly.
"""

from __future__ import annotations

import json
import os
import shutil
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from factorlearn import io as rio  # noqa: E402
from factorlearn.datagen import GenSpec, generate  # noqa: E402
from factorlearn.datasets import ingest_csv, load_dataset, save_dataset  # noqa: E402
from factorlearn.metadata import materialize  # noqa: E402
from factorlearn.sparse import SparseMatrix  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "formats")


def mats():
    rng = np.random.default_rng(3)
    a = rng.random((7, 5)) * (rng.random((7, 5)) < 0.5)
    a[2, :] = 0.0                                  # empty row
    a[0, 0] = 1.0 / 3.0                            # needs 17 digits
    b = -rng.standard_normal((4, 9)) * 1e-7
    return {"sparse": SparseMatrix.from_dense(a), "dense": SparseMatrix.from_dense(b),
            "empty": SparseMatrix.zeros(3, 2)}


def main():
    shutil.rmtree(OUT, ignore_errors=True)
    os.makedirs(OUT)
    exp = {}
    for name, m in mats().items():
        rio.write_matrix_market(os.path.join(OUT, f"{name}.mtx"), m)
        rio.write_binary(os.path.join(OUT, f"{name}.ilg"), m)
        for k in ("indptr", "indices", "data"):
            exp[f"{name}__{k}"] = getattr(m, k)
        exp[f"{name}__shape"] = np.array([m.n_rows, m.n_cols])
    # a saved dataset (outer join, sparse sources)
    ft, params = generate(GenSpec(r_t=60, n_sources=3, sparsity=0.6, join_type="outer", seed=4))
    save_dataset(ft, os.path.join(OUT, "ds_outer"), dataset_id="ds_outer",
                 generator_params=params)
    back, _ = load_dataset(os.path.join(OUT, "ds_outer"))
    exp["ds_outer__T"] = materialize(back).to_dense()
    # CSV star tables (test_datasets.py:21-44 shapes) + union
    with open(os.path.join(OUT, "fact.csv"), "w") as fh:
        fh.write("amount,qty,cust,prod\n10,1,c1,p1\n20,2,c1,p2\n30,3,c2,p1\n40,4,c3,p9\n"
                 "50,5,c2,p3\n")
    with open(os.path.join(OUT, "customers.csv"), "w") as fh:
        fh.write("id,age,income\nc1,25,50\nc2,35,70\nc4,45,90\n")
    with open(os.path.join(OUT, "products.csv"), "w") as fh:
        fh.write("id,price\np1,5\np2,8\np3,9\np4,1.5e-3\n")
    with open(os.path.join(OUT, "u1.csv"), "w") as fh:
        fh.write("a,b\n1,2\n3,4\n")
    with open(os.path.join(OUT, "u2.csv"), "w") as fh:
        fh.write("c\n7\n-0.25\n")
    star = {"fact": {"path": "fact.csv", "keys": {"customers": "cust", "products": "prod"}},
            "dims": {"customers": {"path": "customers.csv", "key": "id"},
                     "products": {"path": "products.csv", "key": "id"}}}
    for jt in ("inner", "left", "outer"):
        m = dict(star, join_type=jt)
        with open(os.path.join(OUT, f"star_{jt}.json"), "w") as fh:
            json.dump(m, fh)
        ft = ingest_csv(m, base_dir=OUT)
        exp[f"star_{jt}__T"] = materialize(ft).to_dense()
        for k, (s, i) in enumerate(zip(ft.sources, ft.indicators)):
            exp[f"star_{jt}__src{k}"] = s.to_dense()
            exp[f"star_{jt}__ind{k}"] = i.matrix.to_dense()
    u = {"join_type": "union", "tables": ["u1.csv", "u2.csv"]}
    with open(os.path.join(OUT, "union.json"), "w") as fh:
        json.dump(u, fh)
    exp["union__T"] = materialize(ingest_csv(u, base_dir=OUT)).to_dense()
    np.savez_compressed(os.path.join(OUT, "expected.npz"), **exp)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
