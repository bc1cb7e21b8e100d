#!/bin/bash
# phase timelines of the config-2 worker step (round 0 and a steady round; modes 0 and 1)
cd "${GRAFT_REPO_ROOT:-.}"; T=${1:-tr}
python tools/trace_step.py 2 0 > gpurun_out/${T}_trace0.log 2>&1
python tools/trace_step.py 2 1 > gpurun_out/${T}_trace1.log 2>&1
