"""Host-side checks that need no GPU: the C-ABI library loads and exports
every entry point `include/fl_b200.h` declares, the ctypes table matches the
header, and the host mirror of the reference interface validates exactly like
the reference (trainers.py:44-64, metadata.py:172-207, ops.py:221-259)."""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fl_b200.h")


def header_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(fl_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    from paper_2502_01985_b200 import _lib
    lib = ctypes.CDLL(_lib.library_path())
    names = header_functions()
    assert len(names) >= 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, f"not exported: {missing}"


def test_ctypes_table_matches_header():
    from paper_2502_01985_b200 import _lib
    assert sorted(_lib.exported_symbols()) == header_functions()


def test_no_device_is_a_loud_error():
    """Without a GPU the product raises instead of falling back to the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2502_01985_b200 import _lib
    with pytest.raises((_lib.BackendUnavailable, _lib.FlError)):
        _lib.device_info(0)


def test_train_config_validation():
    import paper_2502_01985_b200 as fl
    for bad in (dict(iterations=0), dict(learning_rate=0.0), dict(k_clusters=0),
                dict(rank=0), dict(seed=-1)):
        with pytest.raises(fl.ConfigError):
            fl.TrainConfig(**bad)
    with pytest.raises(fl.ConfigError, match="unknown model"):
        fl.train("svm", None, fl.TrainConfig())
    with pytest.raises(fl.ConfigError, match="requires labels"):
        fl.train("linreg", None, fl.TrainConfig())


def test_metadata_validation_matches_reference():
    import paper_2502_01985_b200 as fl
    from paper_2502_01985_b200.metadata import block_mapping, fk_indicator
    s = fl.SparseMatrix.from_dense(np.ones((4, 2)))
    d = fl.SparseMatrix.from_dense(np.ones((2, 2)))
    good = fl.FactorizedTable([s, d], [block_mapping(4, 2, 0), block_mapping(4, 2, 2)],
                              [fk_indicator(4, 4, np.arange(4)), fk_indicator(4, 2, [0, 1, 0, 1])],
                              "inner", 4, 4)
    assert good.validate().ok
    clash = fl.FactorizedTable([s, d], [block_mapping(4, 2, 0), block_mapping(4, 2, 1)],
                               [fk_indicator(4, 4, np.arange(4)),
                                fk_indicator(4, 2, [0, 1, 0, 1])], "inner", 4, 4)
    with pytest.raises(fl.MetadataError):
        clash.require_valid()


def test_sparse_roundtrip_and_structure_checks():
    import paper_2502_01985_b200 as fl
    a = np.array([[0.0, 1.5], [2.0, 0.0], [0.0, 0.0]])
    m = fl.SparseMatrix.from_dense(a)
    assert m.nnz == 2 and np.array_equal(m.to_dense(), a)
    with pytest.raises(fl.SparseStructureError):
        fl.SparseMatrix(2, 2, [0, 1, 1], [5], [1.0])
