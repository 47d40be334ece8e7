#!/bin/bash
# ncu --set full of one implicit sweep launch (config 3, 4 iterations) with source-level stalls.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r2l}
cat > /tmp/imp_step.py <<'PY'
import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import bte_inputs as bi
from paper_2305_19400_b200 import Solver
p = bi.config3()
p.dt *= 8; p.implicit = 1; p.imp_max_iter = 4; p.imp_tol = 0.0
with Solver.from_problem(p) as sv:
    sv.init_random(p.seed, bi.random_phases(p.seed), p.T_init, 20.0, 0.05)
    sv.step(2)
print("done")
PY
R=gpurun_out/prof_imp_${TAG}_c3
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_sweep_imp -s 2 -c 1 -o $R -f python /tmp/imp_step.py > $R.log 2>&1
python scripts/ncu_summary.py rep $R.ncu-rep --workload "config3_implicit" --dof 4194304000 > $R.json
ncu -i $R.ncu-rep --page source --csv > $R.source.csv 2>/dev/null
rm -f $R.ncu-rep
tail -2 $R.log
