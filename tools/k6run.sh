cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | grep -o '"ms_per_step": [0-9.]*\|"leverage": {"ms": [0-9.]*'
