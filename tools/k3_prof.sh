cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT; mkdir -p gpurun_out/prof
timeout 900 ncu --set full --import-source on --clock-control none -k regex:srht_sampled_kernel -c 1 -o gpurun_out/prof/k3 \
  python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/prof/k3.log 2>&1
echo "ncu exit $?"
