#!/bin/bash
# ncu --set full (+ source view) of the hot kernels: config 3 / config 4 sweep, demo sweep and Newton.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r3}
declare -A DOF=( [2]=230400000 [3]=4194304000 [4]=2000000000 [6]=15840000 [7]=460800000 [8]=3145728000 [10]=5280000 )
declare -A WL=( [2]=config2_2d_si_120x120x400x40 [3]="config3_3d_si_64^3x400x40" [4]="config4_3d_si_100^3x400x40" [6]=demo_2d_si_120x120x20x55 [7]=u2_tri_28800x400x40 [8]=u3_tet_196608x400x40 [10]=fig9_2d_si_40x120x20x55 )
for CK in ${CKS:-3:sweep 6:sweep 6:newton}; do
  CFG=${CK%%:*}; K=${CK##*:}
  R=gpurun_out/prof_${K}_${TAG}_c${CFG}
  SKIP=3; [ $CFG = 4 ] && [ $K = sweep ] && SKIP=9
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_${K} -s $SKIP -c 1 \
    -o $R -f python scripts/prof_step.py --config $CFG --warmup 3 --steps 1 > $R.log 2>&1
  python scripts/ncu_summary.py rep $R.ncu-rep --workload "${WL[$CFG]}" --dof ${DOF[$CFG]} > $R.json
  ncu -i $R.ncu-rep --page source --csv > $R.src.csv 2>/dev/null
  rm -f $R.ncu-rep
done
du -sh gpurun_out
