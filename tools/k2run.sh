cd $GRAFT_REPO_ROOT
export PYTHONPATH=$GRAFT_REPO_ROOT
for a in 1 2 3; do
LVSK_K2_APPLY=$a timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | grep -o '"sketch": {"ms": [0-9.]*'
done
