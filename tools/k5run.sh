cd $GRAFT_REPO_ROOT
export PYTHONPATH=$GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "bf16_leverage or c5_shaped" 2>&1 | tail -3
timeout 300 python tools/k5bf16_time.py 8000000 2>&1 | tail -4
