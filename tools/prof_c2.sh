cd $GRAFT_REPO_ROOT
export PYTHONPATH=$GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof3
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"leverage_v2_kernel|hashed_gather_bulk" -c 2 -o gpurun_out/prof3/c2 python bench.py --config c2 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/prof3/ncu_c2.log 2>&1; echo "c2 $?"
