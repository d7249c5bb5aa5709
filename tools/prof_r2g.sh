# session-5: full-set captures with source for the SASS-level stall view (K2, K1, K5, K3)
cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT; mkdir -p gpurun_out/prof7
timeout 900 ncu --set full --import-source on --clock-control none -k regex:csr_sketch_kernel -c 1 -o gpurun_out/prof7/k2 python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu --inflight 1 > /dev/null 2>&1; echo "k2 $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:hashed_gather_bulk_kernel -c 1 -o gpurun_out/prof7/k1 python bench.py --config c2 --steps 1 --warmup 1 --no-e2e --no-cpu --inflight 1 > /dev/null 2>&1; echo "k1 $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:leverage_v2_kernel -c 1 -o gpurun_out/prof7/k5 python bench.py --config c2 --steps 1 --warmup 1 --no-e2e --no-cpu --inflight 1 > /dev/null 2>&1; echo "k5 $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:srht_sampled_kernel -c 1 -o gpurun_out/prof7/k3 python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu --inflight 1 > /dev/null 2>&1; echo "k3 $?"
