"""CPU ORACLE for the run metrics / raw constraint checks — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may use this module.
numpy restatement of the reference ``trajopt.bench.metrics`` (bench/metrics.py:26-95) over a batch of
trajectories, with the obstacle tracks of ``bench.scenarios.predict_obstacles`` (scenarios.py:118-127).
Pinned against golden vectors of the live reference (tests/golden/metrics.npz, tests/test_oracle_metrics.py).
"""

from __future__ import annotations

import numpy as np


def scaled_distances(pos, t, centers, velocities, a, b, dim):
    """metrics.py:55-67 for one trajectory: (n_o, n_p) ellipsoidal distances."""
    tau = t - t[0]  # predict_obstacles with t_now = 0 (scenarios.py:125)
    out = np.empty((len(a), pos.shape[0]))
    for j in range(len(a)):
        cen = centers[j][None, :] + velocities[j][None, :] * tau[:, None]
        delta = pos - cen
        if dim == 3:
            quad = delta[:, 0] ** 2 / a[j] ** 2 + delta[:, 1] ** 2 / a[j] ** 2 + delta[:, 2] ** 2 / b[j] ** 2
        else:
            quad = delta[:, 0] ** 2 / a[j] ** 2 + delta[:, 1] ** 2 / b[j] ** 2
        out[j] = np.sqrt(quad)
    return out


def metrics(pos, acc, t, centers, velocities, a, b, dim, desired=None, margin=0.0):
    """(smoothness, tracking, arc_length, worst, min_clearance) of one trajectory (metrics.py:26-95)."""
    smoothness = float(np.sum(acc**2))
    tracking = 0.0 if desired is None else float(np.sum((pos - desired) ** 2))
    arc = float(np.sum(np.linalg.norm(np.diff(pos, axis=0), axis=1)))
    if len(a) == 0:
        return smoothness, tracking, arc, -np.inf, np.inf
    d = scaled_distances(pos, t, centers, velocities, a, b, dim)
    worst = float(np.max(1.0 + margin - d))
    semi = np.minimum(a, b)[:, None]
    clear = float(np.min((d - 1.0) * semi))
    return smoothness, tracking, arc, worst, clear
