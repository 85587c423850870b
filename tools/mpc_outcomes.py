"""Outcome mix of the receding-horizon fleet for a few field densities / step budgets (diagnostic)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_10731_b200 import scenarios  # noqa: E402
from paper_2408_10731_b200.bench import scenarios as SC  # noqa: E402
from paper_2408_10731_b200.mpc import MpcFleet  # noqa: E402

B = 256
for n_o, budget, steps in ((50, 40, 30), (50, 100, 30), (20, 40, 30), (10, 40, 30), (20, 100, 40), (50, 40, 60)):
    specs = scenarios.flow3d_obstacles(n_o)
    starts, goals = scenarios.flow3d_endpoints(range(B))
    sc = SC.Scenario(kind="dynamic-flow", dim=3, horizon=SC.Horizon(t0=0.0, tf=10.0, n_p=100),
                     robot=SC.RobotSpec(shape=[0.0, 0.0], v_max=3.0, a_max=3.0),
                     obstacles=[SC.ScenarioObstacle(a=o.a, b=o.b, center=[float(x) for x in o.center],
                                                    velocity=[float(x) for x in o.velocity]) for o in specs],
                     boundary=SC.Boundary(start=[0.0, 0.0, 0.0], goal=[12.0, 0.0, 0.0]), seed=0)
    fr = MpcFleet(sc, starts, goals, step_budget=budget).run(steps, early_exit=False)
    f = fr.flags
    end = np.array([fr.trace[i, int(fr.n_trace[i]) - 1] for i in range(B)])
    print(f"n_o {n_o} budget {budget} steps {steps}: collided {int((f == 1).sum())} reached {int((f == 2).sum())} "
          f"driving {int((f == 0).sum())}; median final x {np.median(end[:, 0]):.2f}")
