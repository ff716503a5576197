"""RBCM / CSV matrix files and RBCI index files (reference dataset.py:61-108, rbc.py:228-322).

Fixtures in tests/golden/files/ were written by the REFERENCE (tests/golden/make_golden_files.py).  CPU tests:
read them, write them back byte for byte, and the reference's own format tests (test_dataset.py:16-70,
test_rbc.py:205-258).  GPU tests: this package's builds serialise to the reference's bytes, and a loaded index
searches like a freshly built one.
"""

import dataclasses
import os
import struct

import numpy as np
import pytest

import paper_1103_2635_b200 as rbc

FILES = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "files")
MATRIX = dict(n=400, d=6, seed=5, n_clusters=4, cluster_sigma=0.05)  # make_golden_files.MATRIX


def _golden(name):
    return os.path.join(FILES, name)


def _bytes(path):
    with open(path, "rb") as fh:
        return fh.read()


@pytest.fixture(scope="module")
def data():
    m = MATRIX
    return rbc.gen_synthetic("clusters", m["n"], m["d"], m["seed"], n_clusters=m["n_clusters"],
                             cluster_sigma=m["cluster_sigma"])


@pytest.fixture
def random_matrix():
    rng = np.random.default_rng(3)
    return rbc.DataMatrix((rng.random((100, 8), dtype=np.float32) - 0.5) * 100)


# ---- matrices -------------------------------------------------------------------------------------------------

def test_reference_rbcm_reads_and_rewrites_identically(data, tmp_path):
    m = rbc.load_matrix(_golden("clusters.rbcm"))
    assert np.array_equal(m.values.view(np.uint32), data.values.view(np.uint32))
    rbc.save_matrix(m, tmp_path / "m.rbcm")
    assert _bytes(tmp_path / "m.rbcm") == _bytes(_golden("clusters.rbcm"))


def test_reference_csv_reads_and_rewrites_identically(data, tmp_path):
    m = rbc.load_matrix(_golden("clusters.csv"), "csv")
    assert np.array_equal(m.values.view(np.uint32), data.values.view(np.uint32))
    rbc.save_matrix(m, tmp_path / "m.csv", "csv")
    assert _bytes(tmp_path / "m.csv") == _bytes(_golden("clusters.csv"))


def test_binary_roundtrip_bit_exact(tmp_path, random_matrix):
    rbc.save_matrix(random_matrix, tmp_path / "m.rbcm", "binary")
    back = rbc.load_matrix(tmp_path / "m.rbcm", "binary")
    assert (back.n, back.d) == (100, 8) and np.array_equal(back.values, random_matrix.values)


def test_csv_roundtrip_and_decode(tmp_path, random_matrix):
    rbc.save_matrix(random_matrix, tmp_path / "m.csv", "csv")
    assert np.array_equal(rbc.load_matrix(tmp_path / "m.csv", "csv").values, random_matrix.values)
    (tmp_path / "two.csv").write_text("1.0,2.0\n3.0,4.0\n")
    two = rbc.load_matrix(tmp_path / "two.csv", "csv")
    assert np.array_equal(two.values, np.array([[1, 2], [3, 4]], np.float32))


def test_binary_decode_example(tmp_path):
    (tmp_path / "two.rbcm").write_bytes(b"RBCM" + struct.pack("<III", 1, 2, 2) + np.array([0, 0, 3, 4], "<f4").tobytes())
    m = rbc.load_matrix(tmp_path / "two.rbcm")
    assert (m.n, m.d) == (2, 2) and np.array_equal(m.values, np.array([[0, 0], [3, 4]], np.float32))


@pytest.mark.parametrize("blob,exc", [
    (b"NOPE" + b"\x00" * 12, rbc.FormatError),
    (b"RBCM" + struct.pack("<III", 2, 1, 1) + b"\x00" * 4, rbc.FormatError),
    (b"RBCM" + struct.pack("<III", 1, 0, 3), rbc.FormatError),
    (b"RBCM" + struct.pack("<II", 1, 1), OSError),
    (b"RBCM" + struct.pack("<III", 1, 2, 2) + b"\x00" * 8, OSError),
    (b"RBCM" + struct.pack("<III", 1, 1, 2) + np.array([1.0, np.nan], "<f4").tobytes(), rbc.DataError),
])
def test_bad_matrix_files(tmp_path, blob, exc):
    (tmp_path / "bad.rbcm").write_bytes(blob)
    with pytest.raises(exc):
        rbc.load_matrix(tmp_path / "bad.rbcm")


def test_matrix_path_and_format_errors(tmp_path, random_matrix):
    with pytest.raises(OSError):
        rbc.save_matrix(random_matrix, tmp_path / "missing" / "m.rbcm")
    with pytest.raises(ValueError):
        rbc.save_matrix(random_matrix, tmp_path / "m.x", "parquet")
    with pytest.raises(ValueError):
        rbc.load_matrix(tmp_path / "m.x", "parquet")
    (tmp_path / "bad.csv").write_text("1.0,x\n")
    with pytest.raises(rbc.FormatError):
        rbc.load_matrix(tmp_path / "bad.csv", "csv")


# ---- indexes --------------------------------------------------------------------------------------------------

@pytest.mark.parametrize("name", ["exact_l2.rbci", "one_shot_l1.rbci"])
def test_reference_rbci_reads_and_rewrites_identically(name, data, tmp_path):
    idx = rbc.load_index(_golden(name))
    assert np.array_equal(idx.data.values, data.values)
    rbc.save_index(idx, tmp_path / name)
    assert _bytes(tmp_path / name) == _bytes(_golden(name))


def test_loaded_exact_index_fields():
    idx = rbc.load_index(_golden("exact_l2.rbci"))
    assert isinstance(idx, rbc.RbcExactIndex)
    assert idx.metric == rbc.MetricSpec("l2", 6)
    assert idx.reps.sampling_mode == rbc.BERNOULLI and idx.reps.seed == 0
    # sorted representatives, each first in its own list at distance 0; the lists partition the ids
    assert np.all(np.diff(idx.reps.rep_ids) > 0)
    assert all(ids[0] == r and dd[0] == 0 for r, ids, dd in zip(idx.reps.rep_ids, idx.list_ids, idx.list_dists))
    assert np.array_equal(np.sort(np.concatenate(idx.list_ids)), np.arange(400))
    assert all(a.dtype == np.int64 for a in idx.list_ids) and all(a.dtype == np.float32 for a in idx.list_dists)
    assert np.array_equal(idx.radii, np.array([a.max() if len(a) else 0 for a in idx.list_dists], np.float32))


def test_loaded_one_shot_index_fields():
    idx = rbc.load_index(_golden("one_shot_l1.rbci"))
    assert isinstance(idx, rbc.RbcOneShotIndex)
    assert idx.metric == rbc.MetricSpec("l1", 6) and idx.s == 15
    assert idx.reps.sampling_mode == rbc.FIXED_COUNT and idx.reps.seed == 3
    assert idx.list_ids.shape == (idx.reps.size, 15) and idx.list_ids.dtype == np.int64
    assert np.array_equal(idx.reps.rep_ids, rbc.sample_representatives(400, 15, 3, rbc.FIXED_COUNT).rep_ids)


def test_large_seed_survives(tmp_path):
    idx = rbc.load_index(_golden("exact_l2.rbci"))
    idx = dataclasses.replace(idx, reps=rbc.RepSet(idx.reps.rep_ids, rbc.BERNOULLI, (37 << 40) + 123))
    rbc.save_index(idx, tmp_path / "seed.rbci")
    assert rbc.load_index(tmp_path / "seed.rbci").reps.seed == (37 << 40) + 123


@pytest.mark.parametrize("mutate,exc", [
    (lambda b: b"WHAT" + b[4:], rbc.FormatError),
    (lambda b: b[:4] + struct.pack("<I", 2) + b[8:], rbc.FormatError),
    (lambda b: b[:8] + struct.pack("<I", 7) + b[12:], rbc.FormatError),
    (lambda b: b[:len(b) - 100], OSError),
    (lambda b: b[:30], OSError),
])
def test_bad_index_files(tmp_path, mutate, exc):
    (tmp_path / "bad.rbci").write_bytes(mutate(_bytes(_golden("exact_l2.rbci"))))
    with pytest.raises(exc):
        rbc.load_index(tmp_path / "bad.rbci")


# ---- GPU: this package's builds produce the reference's files ------------------------------------------------

@pytest.mark.gpu
def test_gpu_exact_build_serialises_to_reference_bytes(data, tmp_path):
    idx = rbc.build_exact(data, 20, rbc.MetricSpec("l2", 6), seed=0)
    assert np.array_equal(idx.reps.rep_ids, rbc.load_index(_golden("exact_l2.rbci")).reps.rep_ids)
    rbc.save_index(idx, tmp_path / "e.rbci")
    assert _bytes(tmp_path / "e.rbci") == _bytes(_golden("exact_l2.rbci"))


@pytest.mark.gpu
def test_gpu_one_shot_build_serialises_to_reference_bytes(data, tmp_path):
    idx = rbc.build_one_shot(data, 15, 15, rbc.MetricSpec("l1", 6), seed=3, mode=rbc.FIXED_COUNT)
    rbc.save_index(idx, tmp_path / "o.rbci")
    assert _bytes(tmp_path / "o.rbci") == _bytes(_golden("one_shot_l1.rbci"))


@pytest.mark.gpu
@pytest.mark.parametrize("k", [1, 5])
def test_gpu_loaded_index_searches_like_built(data, k):
    q = rbc.gen_synthetic("clusters", 64, 6, 17, n_clusters=4, cluster_sigma=0.05).values
    built = rbc.build_exact(data, 20, rbc.MetricSpec("l2", 6), seed=0)
    loaded = rbc.load_index(_golden("exact_l2.rbci"))
    (r0, s0), (r1, s1) = rbc.exact_query_batch(built, q, k=k), rbc.exact_query_batch(loaded, q, k=k)
    for a, b in zip(r0, r1):
        assert np.array_equal(a.ids, b.ids) and np.array_equal(a.dists.view(np.uint32), b.dists.view(np.uint32))
    assert s0 == s1
    o_built = rbc.build_one_shot(data, 15, 15, rbc.MetricSpec("l1", 6), seed=3, mode=rbc.FIXED_COUNT)
    o_loaded = rbc.load_index(_golden("one_shot_l1.rbci"))
    (r0, s0), (r1, s1) = rbc.one_shot_query_batch(o_built, q, k=k), rbc.one_shot_query_batch(o_loaded, q, k=k)
    for a, b in zip(r0, r1):
        assert np.array_equal(a.ids, b.ids) and np.array_equal(a.dists.view(np.uint32), b.dists.view(np.uint32))
    assert s0 == s1


def test_random_project_matches_reference_fixture():
    """Same seed, same f64 product: equal to the reference's projection of the fixture matrix."""
    m = rbc.load_matrix(_golden("clusters.rbcm"))
    want = rbc.load_matrix(_golden("random_project_3_8.rbcm")).values
    assert np.array_equal(rbc.random_project(m, 3, 8).values.view(np.uint32), want.view(np.uint32))


def test_random_project_errors():
    m = rbc.DataMatrix(np.ones((4, 3), np.float32))
    with pytest.raises(ValueError):
        rbc.random_project(m, 0, 1)
    with pytest.raises(ValueError):
        rbc.random_project(m, 4, 1)
    with pytest.raises(ValueError):
        rbc.random_project(m, 2, 1, projection=np.ones((2, 2)))
    p = np.eye(3)[:, :2]
    assert np.array_equal(rbc.random_project(m, 2, 1, projection=p).values, np.full((4, 2), 1 / np.sqrt(2), np.float32))
