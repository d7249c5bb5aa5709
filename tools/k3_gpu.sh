cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -k "srht or c3 or variant" 2>&1 | tail -3
timeout 300 python tools/srht_time.py 2>&1 | tail -4
LVSK_SRHT_REGS=1 timeout 300 python tools/srht_time.py 2>&1 | tail -4
timeout 600 python bench.py --config c3 --steps 20 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | grep -o '"ms_per_step": [0-9.]*\|"sketch": {[^}]*}'
