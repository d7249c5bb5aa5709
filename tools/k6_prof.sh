cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT; mkdir -p gpurun_out/prof
timeout 900 ncu --set full --import-source on --clock-control none -k regex:csr_rowsumsq_tc -c 1 -o gpurun_out/prof/k6tc \
  python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/prof/k6tc.log 2>&1
echo "ncu exit $?"
