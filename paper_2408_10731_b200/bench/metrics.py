"""``trajopt.bench.metrics`` drop-in: the GPU implementations live in ``paper_2408_10731_b200.metrics``."""

from ..metrics import RunMetrics, check_collision_free, clearance_lower_bound, eval_metrics, validate_batch  # noqa: F401

__all__ = ["RunMetrics", "eval_metrics", "check_collision_free", "clearance_lower_bound", "validate_batch"]
