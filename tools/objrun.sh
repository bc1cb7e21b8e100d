cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -3
python bench.py --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['roofline']['mean_launch_ms'], d['objective_pass']['ms'], d['e2e']['ms_per_step'])"
