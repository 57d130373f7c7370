"""Golden feature vectors for the cost-estimator corpus,
made by the REAL reference.  Run in the build container:

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_features_golden.py

For every golden table (tests/golden/*.npz, built by make_golden.py) it
rebuilds the table with the reference's own classes, then records the
reference's `extract_features` (features.py:88-121) for all four models at
two training configurations and two hardware specs, and its TR&FR decision
(`estimator.baseline_tr_fr_table`).  Output: features.npz next to this file.
"""

from __future__ import annotations

import glob
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from factorlearn.cost import HardwareSpec  # noqa: E402
from factorlearn.estimator import baseline_tr_fr_table  # noqa: E402
from factorlearn.features import DatasetProfile, extract_features  # noqa: E402
from factorlearn.metadata import FactorizedTable, IndicatorMatrix, MappingMatrix  # noqa: E402
from factorlearn.sparse import SparseMatrix  # noqa: E402
from factorlearn.trainers import TrainConfig  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
CFGS = [(20, 4, 2), (7, 3, 5)]                 # (iterations, k, rank)
HWS = [(148, 6.5533e12), (8, 2.0e10)]          # (parallelism, bytes/s)
MODELS = ("linreg", "logreg", "kmeans", "gnmf")


def ref_table(path):
    raw = np.load(path)
    meta = json.loads(str(raw["meta"]))
    r_t, c_t = meta["r_T"], meta["c_T"]
    srcs, maps, inds = [], [], []
    for k in range(meta["n_sources"]):
        s = raw[f"src{k}"]
        srcs.append(SparseMatrix.from_dense(s))
        mst = raw[f"map_sel_t{k}"]
        ok = mst >= 0
        maps.append(MappingMatrix(SparseMatrix.from_coo(
            c_t, s.shape[1], mst[ok], np.nonzero(ok)[0], np.ones(int(ok.sum())))))
        sel = raw[f"ind_sel{k}"]
        rows = np.nonzero(sel >= 0)[0]
        inds.append(IndicatorMatrix(SparseMatrix.from_coo(
            r_t, s.shape[0], rows, sel[rows], np.ones(rows.size))))
    return FactorizedTable(srcs, maps, inds, meta["join_type"], r_t, c_t)


def main():
    out = {}
    names = []
    for path in sorted(glob.glob(os.path.join(HERE, "*.npz"))):
        name = os.path.basename(path)[:-4]
        if name == "features":
            continue
        ft = ref_table(path)
        prof = DatasetProfile.from_table(ft)
        feats = []
        for it, k, rank in CFGS:
            cfg = TrainConfig(iterations=it, k_clusters=min(k, ft.r_T),
                              rank=min(rank, ft.r_T, ft.c_T))
            for par, bw in HWS:
                hw = HardwareSpec(par, bw)
                for m in MODELS:
                    feats.append(extract_features(prof, m, cfg, hw))
        out[f"{name}__features"] = np.stack(feats)
        out[f"{name}__tr_fr"] = np.array(baseline_tr_fr_table(ft))
        names.append(name)
    out["names"] = np.array(names)
    out["cfgs"] = np.array(CFGS)
    out["hws"] = np.array(HWS)
    np.savez_compressed(os.path.join(HERE, "features.npz"), **out)
    print("wrote", len(names), "tables")


if __name__ == "__main__":
    main()
