#!/bin/bash
# A/B of library variants on the grid-wide path (round 0 of configs 4 and 5 at prof_wide.py sizes):
# tools/wide_ab.sh TAG lib1.so|main ...   -> per-kernel launch tables
cd "${GRAFT_REPO_ROOT:-.}"; T=$1; shift
for v in "$@"; do
  nm=$(basename $v .so)
  if [ "$v" = main ]; then unset HPCG_LIB_OVERRIDE; else export HPCG_LIB_OVERRIDE=$PWD/$v; fi
  for c in 5 4; do
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_${nm}_$c.csv python tools/prof_wide.py $c 1 > /dev/null 2>&1
    echo "== $nm config $c"; python tools/launch_summary.py gpurun_out/${T}_${nm}_$c.csv 6
  done
done
