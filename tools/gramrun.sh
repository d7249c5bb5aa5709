cd $GRAFT_REPO_ROOT
export PYTHONPATH=$GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "kg_ or kf_ or fold or jl_" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_configs.py -q -x -k "c4" 2>&1 | tail -3
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | grep -o '"ms_per_step": [0-9.]*\|"stages_ms": {[^}]*}[^}]*}[^}]*}'
