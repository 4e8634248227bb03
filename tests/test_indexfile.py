"""Index file format (grid.py:204-277): byte-identical with files the
reference itself wrote (tests/golden/index_*.ghn, make_golden.py)."""
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2004_02290_b200.indexfile import FIELDS, MAGIC, read_index_arrays

REF_FILES = ["index_fit_int.ghn", "index_cfg0_str.ghn"]


@pytest.mark.parametrize("name", REF_FILES)
def test_reference_file_parses(name):
    header, arr = read_index_arrays(os.path.join(GOLDEN, name))
    assert header["version"] == 1 and header["metric"] == "euclidean"
    n, d = arr["coords"].shape
    assert arr["order"].shape == (n,) and sorted(arr["order"].tolist()) == list(range(n))
    assert arr["offsets"][0] == 0 and arr["offsets"][-1] == n
    assert arr["cell_ids"].shape == (arr["offsets"].size - 1, d)


def test_bad_magic_rejected(tmp_path):
    p = tmp_path / "junk.ghn"
    p.write_bytes(b"not an index")
    with pytest.raises(ValueError):
        read_index_arrays(p)


@pytest.mark.gpu
@pytest.mark.parametrize("name", REF_FILES)
def test_save_matches_reference_bytes(name, tmp_path):
    import paper_2004_02290_b200 as ghn

    path = os.path.join(GOLDEN, name)
    _, arr = read_index_arrays(path)
    labels = arr["labels"].tolist()
    params = ghn.GridParams(arr["widths"], arr["origin"], arr["splits"])
    if name == "index_cfg0_str.ghn":
        X = np.load(os.path.join(GOLDEN, "index_cfg0_str_X.npy"))        # float32 data, upcast by the reference
    else:
        X = arr["coords"]
    index = ghn.build(ghn.points_from_arrays(np.asarray(X, dtype=np.float64), labels), params=params)
    out = tmp_path / "ours.ghn"
    ghn.save_index(index, out)
    assert out.read_bytes() == open(path, "rb").read()


@pytest.mark.gpu
@pytest.mark.parametrize("name", REF_FILES)
def test_load_save_roundtrip_and_queries(name, tmp_path):
    import oracle
    import paper_2004_02290_b200 as ghn

    path = os.path.join(GOLDEN, name)
    loaded = ghn.load_index(path)
    out = tmp_path / "again.ghn"
    ghn.save_index(loaded, out)
    assert out.read_bytes() == open(path, "rb").read()
    _, arr = read_index_arrays(path)
    ref = oracle.COracle(arr["coords"], arr["widths"])
    Q = arr["coords"][:25] + 0.01
    dist, idx, stats = ghn.knn_query_batch(loaded, Q, 3, "guaranteed")
    keys, ridx, rstats = ref.query(Q, 3, "guaranteed")
    assert np.array_equal(idx.cpu().numpy(), ridx) and np.array_equal(stats.cpu().numpy(), rstats)
