"""Native greedy region growing (swb_build_aggregation, host code in the
library) vs the reference's cluster ids (aggregation.py:89-127).  CPU only:
the function works on host buffers."""

import numpy as np
import pytest

from conftest import load_golden
from paper_1607_04174_b200 import types as T
from paper_1607_04174_b200.aggregation import build_aggregation


@pytest.mark.parametrize("tag", ["2", "3"])
def test_build_aggregation_matches_reference(tag):
    z = load_golden("aggregation")
    dims = tuple(int(d) for d in z["dims" + tag])
    pri = T.ProbabilityField(dims, z["pri" + tag])
    agg = build_aggregation(pri, int(z["radius" + tag]), float(z["tol" + tag]))
    np.testing.assert_array_equal(agg.cluster_ids, z["cid" + tag])
    assert agg.n_super == int(z["nsup" + tag])


@pytest.mark.parametrize("radius,tol", [(0, 1.0), (3, 0.0), (50, 10.0), (2, 0.2)])
def test_build_aggregation_edge_cases_vs_oracle(radius, tol):
    from oracle import rw_oracle as O
    rng = np.random.default_rng(radius)
    dims = (7, 6, 5)
    p = rng.random((210, 4))
    p /= p.sum(axis=1, keepdims=True)
    agg = build_aggregation(T.ProbabilityField(dims, p), radius, tol)
    cid, ns = O.build_aggregation(p, dims, radius, tol)
    np.testing.assert_array_equal(agg.cluster_ids, cid)
    assert agg.n_super == ns
