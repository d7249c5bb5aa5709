cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT; mkdir -p gpurun_out/prof9
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:gaussian_tc_pair_kernel -c 1 -o gpurun_out/prof9/k4 python bench.py --config c5 --steps 1 --warmup 1 --no-e2e --no-cpu --inflight 1 > gpurun_out/prof9/k4.log 2>&1; echo "k4 $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gram_i8_kernel -c 1 -o gpurun_out/prof9/kg python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu --inflight 1 > /dev/null 2>&1; echo "kg $?"
