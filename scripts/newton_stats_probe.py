import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import bte_inputs as bi
from paper_2305_19400_b200 import Solver
for cfg in (3, 6):
    p = bi.config3() if cfg == 3 else bi.config_demo()
    with Solver.from_problem(p) as sv:
        sv.init_random(p.seed, bi.random_phases(p.seed), p.T_init, 20.0, 0.05)
        sv.step(5)
        print("after warm-up", cfg, flush=True)
        sv.step(1)
        sv.step(1)
