cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT; mkdir -p gpurun_out/prof
timeout 900 ncu --set full --import-source on --clock-control none -k regex:leverage_v2_kernel -c 1 -o gpurun_out/prof/k5v2 \
  python bench.py --config c2 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/prof/k5v2.log 2>&1
echo "ncu exit $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:hashed_gather_bulk -c 1 -o gpurun_out/prof/k1 \
  python bench.py --config c2 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/prof/k1.log 2>&1
echo "ncu exit $?"
