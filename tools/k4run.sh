cd $GRAFT_REPO_ROOT
export PYTHONPATH=$GRAFT_REPO_ROOT
timeout 300 python tools/k4_time.py 1000000 2>&1 | tail -10
timeout 300 python tools/k4_time.py 8000000 2>&1 | tail -10
