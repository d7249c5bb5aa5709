cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT; mkdir -p gpurun_out/prof8
timeout 900 ncu --set full --import-source on --clock-control none -k regex:csr_rowsumsq_tc2_kernel -c 1 -o gpurun_out/prof8/k6v2b python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu --inflight 1 > /dev/null 2>&1; echo "k6 $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:chol_fold_kernel -c 1 -o gpurun_out/prof8/kf python bench.py --config c2 --steps 1 --warmup 1 --no-e2e --no-cpu --inflight 1 > /dev/null 2>&1; echo "kf $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:argsort_coop_kernel -c 1 -o gpurun_out/prof8/k7 python bench.py --config c2 --steps 1 --warmup 1 --no-e2e --no-cpu --inflight 1 > /dev/null 2>&1; echo "k7 $?"
