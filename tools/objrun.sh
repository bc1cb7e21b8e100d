cd $GRAFT_REPO_ROOT
for v in "" tools/var_TG.so "" tools/var_TG.so; do
  echo "== ${v:-main}"
  for a in --means ""; do HPCG_LIB_OVERRIDE=$v python tools/dbg_obj.py $a 2>&1 | head -1; done
done
HPCG_LIB_OVERRIDE=tools/var_TG.so timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -2
