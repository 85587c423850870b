"""Results-file and trajectory-dump wire formats (reference bench/runner.py:26-38,
247-304).

Byte-compatible with the reference's writers (pinned by ``tests/golden/wire/``): the header row, the column
order, ``repr`` for every float (so identical runs give identical bytes, signed zeros, ``inf`` and denormals
included), ``true``/``false`` for success, integers for seed / iters, and blank cells for the z / psi columns a
trajectory does not have.  ``wall_time_ms`` is the one column that differs between runs.
"""

from __future__ import annotations

import csv
from dataclasses import dataclass
from pathlib import Path

from ..metrics import RunMetrics

__all__ = ["RESULTS_COLUMNS", "RunRecord", "write_trajectory_csv", "write_results_csv", "read_results_csv"]

RESULTS_COLUMNS = ("scenario_id", "solver", "seed", "success", "smoothness", "tracking", "arc_length", "iters",
                   "residual_final", "min_clearance", "wall_time_ms")

# column -> (cell writer, cell reader); every other column is a float written with repr
_TEXT = (str, str)
_INT = (lambda v: str(int(v)), int)
_BOOL = (lambda v: "true" if v else "false", lambda s: s == "true")
_FLOAT = (lambda v: repr(float(v)), float)
_CODEC = {"scenario_id": _TEXT, "solver": _TEXT, "seed": _INT, "iters": _INT, "success": _BOOL}


def _codec(col: str):
    return _CODEC.get(col, _FLOAT)


@dataclass
class RunRecord:
    scenario_id: str
    solver: str
    seed: int
    metrics: RunMetrics
    trajectory_path: str | None = None

    def row(self) -> list:
        fields = dict(vars(self.metrics), scenario_id=self.scenario_id, solver=self.solver, seed=self.seed)
        return [_codec(c)[0](fields[c]) for c in RESULTS_COLUMNS]


def write_trajectory_csv(path, traj, dim: int, psi=None) -> None:
    """Columns t, x, y, z, psi (z blank for planar paths, psi blank when absent)."""
    r = lambda v: repr(float(v))  # noqa: E731
    with open(path, "w", newline="") as fh:
        out = csv.writer(fh)
        out.writerow(["t", "x", "y", "z", "psi"])
        for k in range(len(traj.t)):
            p = traj.pos[k]
            out.writerow([r(traj.t[k]), r(p[0]), r(p[1]), r(p[2]) if dim == 3 else "",
                          "" if psi is None else r(psi[k])])


def write_results_csv(path, records: list, append: bool = True) -> None:
    """One row per record; a header only when the file is new (or append=False)."""
    path = Path(path)
    new_file = not append or not path.exists()
    with open(path, "w" if new_file else "a", newline="") as fh:
        out = csv.writer(fh)
        if new_file:
            out.writerow(RESULTS_COLUMNS)
        out.writerows(rec.row() for rec in records)


def read_results_csv(path) -> list:
    """(scenario_id, solver, seed, RunMetrics) records back from a results file."""
    records = []
    with open(path, newline="") as fh:
        for row in csv.DictReader(fh):
            v = {c: _codec(c)[1](row[c]) for c in RESULTS_COLUMNS}
            m = RunMetrics(**{k: v[k] for k in ("smoothness", "tracking", "arc_length", "success", "iters",
                                                 "residual_final", "min_clearance", "wall_time_ms")})
            records.append(RunRecord(scenario_id=v["scenario_id"], solver=v["solver"], seed=v["seed"], metrics=m))
    return records
