"""Pin the metrics oracle (oracle/metrics.py) against golden vectors of the live reference (bench/metrics.py)."""

import numpy as np
import pytest

from oracle import metrics as OMT


def obstacle_arrays(g, tag, dim):
    o = g[f"{tag}_obs"]
    return o[:, :dim], o[:, dim:2 * dim], o[:, 2 * dim], o[:, 2 * dim + 1]


@pytest.mark.parametrize("tag,dim", [("s3", 3), ("f2", 2)])
def test_metrics_bitexact(golden, tag, dim):
    g = golden("metrics.npz")
    c, v, a, b = obstacle_arrays(g, tag, dim)
    for x, ref in zip(g[f"{tag}_xi"], g[f"{tag}_res"]):
        pos, acc = g[f"{tag}_P"] @ x.T, g[f"{tag}_Pdd"] @ x.T
        sm, tr, arc, w0, cl = OMT.metrics(pos, acc, g[f"{tag}_t"], c, v, a, b, dim, g[f"{tag}_desired"], 0.0)
        w1 = OMT.metrics(pos, acc, g[f"{tag}_t"], c, v, a, b, dim, None, 0.1)[3]
        np.testing.assert_array_equal([sm, tr, arc, cl, w0, float(w0 <= 0), w1, float(w1 <= 0), cl], ref)
