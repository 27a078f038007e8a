"""Dispersion proxy (oracle.py:141-158) and the advisory filter radius
(morton.py:239-245) against reference outputs (tests/golden/dispersion.npz:
the reference's dispersion_stats and the per-point float64 cKDTree values it
is built on)."""

import numpy as np
import pytest

from conftest import load_golden

from paper_2406_02807_b200 import dispersion as D

CASES = ("uniform", "dups", "k2", "cfg1", "tiny")


def test_safe_filter_radius_and_small_clouds():
    assert D.safe_filter_radius(0.02, 0.005) == pytest.approx(0.015)
    assert D.safe_filter_radius(0.01, 0.05) == 0.0
    with pytest.raises(ValueError, match="at least 2 points"):
        D.dispersion_stats(np.zeros((1, 3), np.float32))


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES)
def test_device_nn_and_stats_match_reference(case):
    z = load_golden("dispersion.npz")
    pts = z[f"{case}/points"]
    nn = D.nn_distances(pts)
    assert np.array_equal(nn, z[f"{case}/nn"])  # bit-exact per point
    st = D.dispersion_stats(pts)
    mean, median, p95, count = z[f"{case}/stats"]
    assert (st.mean, st.median, st.p95, st.count) == (mean, median, p95, int(count))
