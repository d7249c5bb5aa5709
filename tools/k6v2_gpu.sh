cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -k "csr or c4" --timeout 200 2>&1 | tail -3
timeout 600 python tools/k6v2_time.py 4000000 4 6 8 10 12 16 2>&1 | tee gpurun_out/k6v2_time.log | grep "v2\|v1"
