cd $GRAFT_REPO_ROOT
export PYTHONPATH=$GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "argsort or order" 2>&1 | tail -2
timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | grep -o '"ms_per_step": [0-9.]*\|"order_ms": [0-9.]*'
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | grep -o '"ms_per_step": [0-9.]*\|"order_ms": [0-9.]*\|"leverage": {"ms": [0-9.]*'
