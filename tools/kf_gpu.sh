cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py -q -x -k "chol or kf or jl_fold or fold_cert or uncertified or pipeline or kg or batch" 2>&1 | tail -3
timeout 300 python tools/kf_time.py 2>&1 | tail -5
timeout 600 python bench.py --config c2 --steps 20 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | grep -o '"ms_per_step": [0-9.]*\|"factor_ms": [0-9.]*\|"latency_ms_per_pass": [0-9.]*'
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | grep -o '"ms_per_step": [0-9.]*\|"factor_ms": [0-9.]*'
