"""eval.py (ball counts, expansion rate, rank error, Claim-1) and report.py rank errors against the reference.

Golden outputs come from the reference itself (tests/golden/make_golden_eval.py); inputs are regenerated here
from the same seeds.  All comparisons are exact (integer counts; float ratios computed from identical counts).
"""

import hashlib
import os

import numpy as np
import pytest

import paper_1103_2635_b200 as rbc
from paper_1103_2635_b200 import eval as ev

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "eval_golden.npz")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


@pytest.fixture(scope="module")
def inputs():
    """Kept in sync with tests/golden/make_golden_eval.py::inputs."""
    data = rbc.gen_synthetic("clusters", 3000, 8, 21, n_clusters=6, cluster_sigma=0.05)
    queries = rbc.gen_synthetic("clusters", 3200, 8, 21, n_clusters=6, cluster_sigma=0.05).values[3000:]
    return data, np.ascontiguousarray(queries)


# ---- argument errors (raised before any device work, so they run on CPU) -------------------------------------

def test_argument_errors(inputs):
    data, queries = inputs
    spec = rbc.MetricSpec("l2", 8)
    with pytest.raises(ValueError):
        rbc.ball_count(data, data.values[0], -1.0, spec)
    with pytest.raises(ValueError):
        rbc.rank_error(data, queries[0], 3000, spec)
    with pytest.raises(ValueError):
        rbc.rank_error(data, queries[0], -1, spec)
    with pytest.raises(ValueError):
        rbc.estimate_expansion_rate(data, spec, 0, 4, 0)
    with pytest.raises(ValueError):
        rbc.estimate_expansion_rate(data, spec, 4, 0, 0)
    with pytest.raises(ValueError):
        rbc.claim1_counts(data, 10, spec, 500, 0, queries=queries)
    with pytest.raises(ValueError):
        rbc.ball_count(data, np.zeros(3, np.float32), 1.0, spec)


def test_threshold_chunk_size_fits_shared_budget():
    for d in (1, 8, 64, 1024):
        nt = ev._max_thresholds(d)
        assert nt >= 1 and 4 * d + 140 * nt + 16 <= 46 * 1024


# ---- parity with the reference ---------------------------------------------------------------------------------

KINDS = ["l2", "l1"]


@pytest.mark.gpu
@pytest.mark.parametrize("kind", KINDS)
def test_ball_count(kind, inputs, gold):
    data, _ = inputs
    spec = rbc.MetricSpec(kind, 8)
    radii = [0.0, 0.01, 0.05, 0.1, 0.3, 1.0, 10.0]
    got = np.array([[rbc.ball_count(data, data.values[c], r, spec) for r in radii] for c in (0, 7, 1234, 2999)])
    assert np.array_equal(got, gold[f"ball_{kind}"])


@pytest.mark.gpu
@pytest.mark.parametrize("kind", KINDS)
def test_estimate_expansion_rate(kind, inputs, gold):
    data, queries = inputs
    spec = rbc.MetricSpec(kind, 8)
    got = []
    for seed, ns, nr, qq in ((0, 20, 8, None), (5, 7, 200, None), (9, 12, 16, queries[:50])):
        e = rbc.estimate_expansion_rate(data, spec, ns, nr, seed, queries=qq)
        got.append([e.c_max, e.c_median, e.samples, e.radii_per_sample, float(e.includes_queries)])
    assert np.array_equal(np.array(got), gold[f"expansion_{kind}"])


@pytest.mark.gpu
@pytest.mark.parametrize("kind", KINDS)
def test_rank_error(kind, inputs, gold):
    data, queries = inputs
    spec = rbc.MetricSpec(kind, 8)
    got = [rbc.rank_error(data, queries[i], rid, spec) for i, rid in ((0, 0), (1, 17), (2, 2999), (3, 1500), (4, 42))]
    assert np.array_equal(np.array(got), gold[f"rank_{kind}"])


@pytest.mark.gpu
@pytest.mark.parametrize("kind", KINDS)
def test_claim1_counts(kind, inputs, gold):
    data, queries = inputs
    spec = rbc.MetricSpec(kind, 8)
    assert np.array_equal(rbc.claim1_counts(data, 60, spec, 40, 3), gold[f"claim1_box_{kind}"])
    assert np.array_equal(rbc.claim1_counts(data, 200, spec, 30, 4, queries=queries), gold[f"claim1_q_{kind}"])
    assert rbc.claim1_trial(data, 60, spec, 40, 3) == float(gold[f"claim1_box_{kind}"].mean())


@pytest.mark.gpu
@pytest.mark.parametrize("kind", KINDS)
def test_baseline_and_rank_errors(kind, inputs, gold):
    data, queries = inputs
    spec = rbc.MetricSpec(kind, 8)
    base = ev.run_baseline(data, queries, spec, 1)
    assert base.top_dists.shape == (200, 512) and base.evals_per_query == 3000
    assert np.array_equal(base.top_dists[:16].view(np.uint32), gold[f"baseline_top16_{kind}"].view(np.uint32))
    assert hashlib.sha256(np.ascontiguousarray(base.top_dists).tobytes()).hexdigest() == str(gold[f"baseline_sha_{kind}"])
    ranks = ev.rank_errors(data, queries, gold[f"rank_ret_{kind}"], base, spec)
    assert np.array_equal(ranks, gold[f"rank_errors_{kind}"])
    assert (ranks >= 512).any() and (ranks[:20] == 0).all()  # both the baseline and the counting path ran


@pytest.mark.gpu
def test_count_within_matches_distance_rows():
    """Closed/strict counts and row maxima against a direct count over the exact distance rows."""
    rng = np.random.default_rng(4)
    for d in (1, 5, 64, 130):
        x = rng.random((2500, d), dtype=np.float32)
        q = rng.random((37, d), dtype=np.float32)
        for kind in KINDS:
            spec = rbc.MetricSpec(kind, d)
            rows = rbc.distance_rows(q, x, spec).astype(np.float64)
            thr = np.sort(rows[:, rng.integers(2500, size=9)], axis=1)
            thr[:, 0] = rows[:, 5]  # a threshold equal to an actual distance: < vs <= differ
            for strict in (False, True):
                got, mx = ev.count_within(q, x, spec, thr, strict, want_max=True)
                want = ((rows[:, None, :] < thr[:, :, None]) if strict else (rows[:, None, :] <= thr[:, :, None])).sum(-1)
                assert np.array_equal(got, want)
                assert np.array_equal(mx, rows.max(1).astype(np.float32))
