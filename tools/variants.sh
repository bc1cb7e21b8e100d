#!/bin/bash
# bench.py under environment variants (diagnostic switches): one JSON line per variant
cd "${GRAFT_REPO_ROOT:-.}"; T=${1:-var}; shift
for v in "$@"; do
  env $v python bench.py --steps 8 --warmup 3 --no-cpu --no-e2e --no-configs > gpurun_out/${T}_$(echo $v | tr '= ' '__').log 2>&1
done
