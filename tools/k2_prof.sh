# ncu full set + source of K2 (csr_sketch_kernel) on C4, one launch
cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT; mkdir -p gpurun_out/prof
timeout 900 ncu --set full --import-source on --clock-control none -k regex:csr_sketch_kernel -c 1 -o gpurun_out/prof/k2v3 \
  python tools/k2_time.py 1000000 > gpurun_out/prof/k2v3.log 2>&1
echo "ncu exit $?"; tail -3 gpurun_out/prof/k2v3.log
