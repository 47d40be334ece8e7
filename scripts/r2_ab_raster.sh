#!/bin/bash
# A/B of the 3-D sweep's column order (BTE_RASTER strips), segment count
# (BTE_SEGS) and L2 policies (BTE_L2HINT) on configs 4 and 3: bench lines +
# per-launch DRAM bytes from ncu (one sweep launch each).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r2c}
OUT=gpurun_out/ab_${TAG}.jsonl
: > $OUT
VARS=${VARS:-"BTE_RASTER=0 BTE_L2HINT=1 BTE_L2HINT=2 BTE_RASTER=16 BTE_RASTER=25 BTE_RASTER=16,BTE_SEGS=3 BTE_RASTER=25,BTE_SEGS=3 BTE_RASTER=32,BTE_SEGS=3 BTE_RASTER=16,BTE_SEGS=2 BTE_RASTER=32,BTE_SEGS=2 BTE_RASTER=50,BTE_SEGS=2"}
for CFG in ${CFGS:-4 3}; do
  for V in $VARS; do
    ENVS=$(echo $V | tr ',' ' ')
    L=$(env $ENVS timeout 300 python bench.py --config $CFG --steps 10 --repeats 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null)
    env $ENVS timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
      -k regex:k_sweep -s $([ $CFG = 4 ] && echo 9 || echo 2) -c 1 --csv python scripts/prof_step.py --config $CFG --warmup 2 --steps 1 > /tmp/ncu_ab.csv 2>/dev/null
    python - "$CFG" "$V" "$L" >> $OUT <<'PY'
import csv, io, json, sys
cfg, var, line = sys.argv[1], sys.argv[2], sys.argv[3]
txt = open('/tmp/ncu_ab.csv').read()
i = txt.find('"ID"')
m = {}
if i >= 0:
    for r in csv.DictReader(io.StringIO(txt[i:])):
        m[r["Metric Name"]] = (float(r["Metric Value"].replace(",", "")), r["Metric Unit"])
dof = {"3": 4194304000, "4": 2000000000}[cfg]
sc = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}
def val(k):
    v = m.get(k)
    return None if v is None else v[0] * sc.get(v[1], 1)
rd, wr, t = val("dram__bytes_read.sum"), val("dram__bytes_write.sum"), val("gpu__time_duration.sum")
out = {"config": cfg, "variant": var}
try:
    d = json.loads(line)
    r = d["roofline"]
    out.update(ms_per_step=d["ms_per_step"], sweep_ms=r["kernel_ms_avg"], frac=r["frac"], sm_mhz=d["clocks"]["sm_mhz"])
except Exception as e:
    out["bench_error"] = str(e)[:200]
if rd is not None and wr is not None:
    out.update(ncu_ms=t * 1e3 if t else None, dram_B_per_dof=(rd + wr) / dof, rd_B_per_dof=rd / dof,
               ncu_TBps=(rd + wr) / t / 1e12 if t else None, ncu_alg_frac=16 * dof / t / 6.54e12 if t else None)
print(json.dumps(out))
PY
  done
done
cat $OUT
