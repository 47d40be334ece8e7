"""Minimal driver for ncu: config N (default 2), device random start, W warm-up
steps then S profiled steps.  Kernel launches per step: [k_diffuse...], k_sweep, k_newton."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bte_inputs as bi  # noqa: E402
from paper_2305_19400_b200 import Solver  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--start", default="random")
ap.add_argument("--tau", type=int, default=0)
a = ap.parse_args()
p = {2: bi.config2, 3: bi.config3, 4: bi.config4, 1: bi.config1, 5: bi.config5, 6: bi.config_demo, 7: bi.config_u2,
     8: bi.config_u3, 9: bi.config_uq, 10: bi.config_fig9, 11: bi.config_u3h}[a.config]()
with Solver.from_problem(p) as sv:
    if a.tau:
        sv.set_tau_mode(a.tau)
    if a.start == "random":
        sv.init_random(p.seed, bi.random_phases(p.seed), p.T_init, 20.0, 0.05)
    sv.step(a.warmup)
    sv.step(a.steps)
print("done", p.name)
