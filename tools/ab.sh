#!/bin/bash
# A/B of library variants on the config-2 bench (dev tool): tools/ab.sh TAG lib1.so [lib2.so ...]
# ("main" = the in-tree libhpcg.so). One JSON line each + the step geometry (HPCG_DEBUG).
cd "${GRAFT_REPO_ROOT:-.}"; T=$1; shift
for v in "$@"; do
  nm=$(basename $v .so)
  if [ "$v" = main ]; then unset HPCG_LIB_OVERRIDE; else export HPCG_LIB_OVERRIDE=$PWD/$v; fi
  HPCG_DEBUG=1 timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu --no-e2e --no-configs > gpurun_out/${T}_$nm.log 2>&1
  python - "$T" "$nm" <<'PY'
import json, sys
t, nm = sys.argv[1:3]
lines = open(f"gpurun_out/{t}_{nm}.log").read().splitlines()
geo = sorted({l for l in lines if l.startswith("[hpcg] step")})
try:
    r = json.loads(lines[-1])
    print(nm, "ms/step %.3f" % r["ms_per_step"], "step launch ms %.4f" % r["roofline"]["mean_launch_ms"],
          "frac %.4f" % r["roofline"]["frac"], "obj GB/s %.0f" % r["objective_pass"]["gbs"], geo[:2])
except Exception as e:
    print(nm, "FAILED", lines[-3:])
PY
done
