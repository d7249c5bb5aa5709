cd $GRAFT_REPO_ROOT
export PYTHONPATH=$GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_bench_multirank.py -q -x -k "k1_folded or hashed or pipeline or c2 or multirank" 2>&1 | tail -2
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu 2>&1 | tail -1 | grep -o '"ms_per_step": [0-9.]*\|"stages_ms": {[^}]*}[^}]*}[^}]*}\|"frac": [0-9.]*'
