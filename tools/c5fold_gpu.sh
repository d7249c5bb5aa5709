cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -k "rank or jl or c5 or topk or spectral or fold" 2>&1 | tail -3
timeout 600 python bench.py --config c5 --steps 10 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | grep -o '"ms_per_step": [0-9.]*\|"factor_ms": [0-9.]*'
