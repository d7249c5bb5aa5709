cd $GRAFT_REPO_ROOT
export PYTHONPATH=$GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "csr" 2>&1 | tail -3
timeout 600 python tools/k6_time.py 2>&1 | tail -4
