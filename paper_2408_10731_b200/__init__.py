"""B200-native batched AM/AL trajectory optimizer (arXiv 2408.10731).

Drop-in for the reference ``trajopt`` package's hot path: the same module
names (``basis``, ``geometry``, ``qpcore``, ``solver_single``, ``solver_batch``,
``solver_priest``, ``solver_multiagent``) and public signatures, with every
per-iteration step executed by hand-written sm_100a CUDA kernels behind the
C-ABI in ``include/trajopt_b200.h``.

    import paper_2408_10731_b200 as trajopt
    sol = trajopt.solver_single.solve_single(problem, params)
    ranked = trajopt.solver_batch.solve_batch_opt(batch_problem, batch_params)
"""

from . import basis, geometry, qpcore, scenarios, solver_batch, solver_multiagent, solver_priest, solver_single  # noqa: F401

__version__ = "0.1.0"

__all__ = ["basis", "geometry", "qpcore", "scenarios", "solver_batch", "solver_multiagent", "solver_priest",
           "solver_single", "__version__"]
