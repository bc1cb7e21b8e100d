#!/bin/bash
# A/B of library variants on the f(C,X) passes (config 2 via prof_obj-like timing, configs 3/4/5):
# tools/obj_ab.sh TAG lib1.so|main ...
cd "${GRAFT_REPO_ROOT:-.}"; T=$1; shift
for v in "$@"; do
  nm=$(basename $v .so)
  if [ "$v" = main ]; then unset HPCG_LIB_OVERRIDE; else export HPCG_LIB_OVERRIDE=$PWD/$v; fi
  echo "== $nm"
  python tools/prof_obj_time.py 2>&1 | tail -1
  for c in 5 4 3; do python tools/prof_cfg_obj.py $c 2>&1 | tail -1; done
done
