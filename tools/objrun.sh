cd $GRAFT_REPO_ROOT
for v in "" tools/var_U4.so tools/var_T1.so; do
  echo "== variant ${v:-main}"
  for a in --means "" --means; do HPCG_LIB_OVERRIDE=$v python tools/dbg_obj.py $a 2>&1 | head -1; done
done
timeout 600 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -2
HPCG_LIB_OVERRIDE=tools/var_U4.so timeout 600 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -2
