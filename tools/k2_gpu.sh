cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -k "csr or c4 or nonfinite" 2>&1 | tail -3
timeout 600 python tools/k2_time.py 2>&1 | tail -12
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | cut -c1-1000
