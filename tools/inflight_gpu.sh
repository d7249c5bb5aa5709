cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
for c in c2 c3 c1; do for f in 2 3 4; do
  echo -n "$c inflight $f: "; timeout 600 python bench.py --config $c --steps 30 --warmup 5 --no-e2e --no-cpu --inflight $f 2>&1 | tail -1 | grep -o '"ms_per_step": [0-9.]*'
done; done
