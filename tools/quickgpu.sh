cd $GRAFT_REPO_ROOT
export PYTHONPATH=$GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "streamed or srht_sampled_vs" 2>&1 | tail -2
LVSK_NVTX=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | cut -c1-200
