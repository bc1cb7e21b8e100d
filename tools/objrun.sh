cd $GRAFT_REPO_ROOT
for c in "" 7 8 10 12; do
  echo "== cluster ${c:-auto}"
  HPCG_CLUSTER=$c HPCG_DEBUG=1 python tools/quick_time.py 2>&1 | grep -E "round [0-3]|cluster" | head -5
done
