cd $GRAFT_REPO_ROOT
export PYTHONPATH=$GRAFT_REPO_ROOT
LVSK_SORT_TRACE=1 timeout 300 python tools/sort_trace.py 2>&1 | tail -12
LVSK_KF_TRACE=1 timeout 300 python tools/kf_trace.py 2>&1 | tail -12
