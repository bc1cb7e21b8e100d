#!/bin/bash
# Dev tool: config-2 bench under pinned worker-step cluster sizes (HPCG_CLUSTER): tools/cluster_sweep.sh TAG 8 9 10 ...
cd "${GRAFT_REPO_ROOT:-.}"; T=$1; shift
for c in "$@"; do
  if [ "$c" = auto ]; then unset HPCG_CLUSTER; else export HPCG_CLUSTER=$c; fi
  HPCG_DEBUG=1 timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu --no-e2e --no-configs > gpurun_out/${T}_c$c.log 2>&1
  python - "$T" "$c" <<'PY'
import json, sys
t, c = sys.argv[1:3]
lines = open(f"gpurun_out/{t}_c{c}.log").read().splitlines()
geo = sorted({l for l in lines if l.startswith("[hpcg] step")})
try:
    r = json.loads(lines[-1])
    print("cluster", c, "ms/step %.3f" % r["ms_per_step"], "step launch ms %.4f" % r["roofline"]["mean_launch_ms"], geo[:1])
except Exception as e:
    print("cluster", c, "FAILED", lines[-3:])
PY
done
