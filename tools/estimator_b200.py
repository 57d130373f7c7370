#!/usr/bin/env python
"""Retrain the reference's factorize-vs-materialize estimator on the B200
corpus and score it.  Build-container tool: it imports
the UNMODIFIED reference (`factorlearn.estimator` / `gbdt`) from
/root/reference as a library, the same way a `factorlearn` user would feed it
a corpus; nothing on the GPU path uses it.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tools/estimator_b200.py \
        profiles/r01_c5_sweep_10M_corpus.csv > profiles/r01_c5_estimator.json

Reports, on a seeded 80/20 split (estimator.split_corpus) and on the whole
corpus with 5-fold cross-validation, the accuracy / F1 / overall speedup
(sum t_mat / sum t_chosen, estimator.evaluate) of: the GBDT retrained on B200
timings, the same GBDT without the hardware feature group, the TR&FR
threshold rule, always-materialize and the oracle.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from factorlearn import estimator as est  # noqa: E402


def score(train, test):
    out = {}
    m = est.fit_estimator(train)
    out["gbdt_b200"] = est.evaluate(est.decide_with_model(m, test), test)
    m2 = est.fit_estimator(train, use_hardware_features=False)
    out["gbdt_no_hw"] = est.evaluate(est.decide_with_model(m2, test), test)
    out["tr_fr"] = est.evaluate(est.decide_recorded_baseline(test), test)
    out["always_materialize"] = est.evaluate(est.decide_always_materialize(test), test)
    out["oracle"] = est.evaluate(est.decide_oracle(test), test)
    return out


def main():
    path = sys.argv[1]
    runs = est.read_corpus(path)
    train, test = est.split_corpus(runs, test_fraction=0.2, seed=0)
    res = {"corpus": os.path.basename(path), "runs": len(runs),
           "factorized_faster": int(sum(r.label for r in runs)),
           "split_80_20": score(train, test)}
    # 5-fold CV (seeded): mean of each policy's metrics
    order = np.random.default_rng(0).permutation(len(runs))
    folds = np.array_split(order, 5)
    cv = {}
    for f in folds:
        te = [runs[i] for i in sorted(f)]
        tr = [runs[i] for i in range(len(runs)) if i not in set(f.tolist())]
        if len({r.label for r in tr}) < 2:
            continue
        for k, v in score(tr, te).items():
            cv.setdefault(k, []).append(v)
    res["cv5_mean"] = {k: {m: float(np.mean([d[m] for d in v])) for m in ("accuracy", "f1",
                                                                            "overall_speedup")}
                       for k, v in cv.items()}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
