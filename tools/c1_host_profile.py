"""Where does solve_single's host time go (C1 converged solve)?"""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_10731_b200 import scenarios, solver_single  # noqa: E402

prob = scenarios.c1_problem()
for _ in range(3):
    solver_single.solve_single(prob, solver_single.SingleParams())
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    solver_single.solve_single(prob, solver_single.SingleParams())
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
