cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
mkdir -p gpurun_out
echo "stream loads:"; timeout 600 python tools/k6v2_time.py 4000000 8 10 12 14 2>&1 | grep v2
echo "L1-allocating M loads:"; LVSK_K6_DBG=4 timeout 600 python tools/k6v2_time.py 4000000 8 10 12 14 16 2>&1 | grep v2
echo "L1-allocating, no walk:"; LVSK_K6_DBG=6 timeout 600 python tools/k6v2_time.py 4000000 8 12 16 2>&1 | grep v2
