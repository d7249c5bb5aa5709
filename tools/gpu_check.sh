cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -25 gpurun_out/pytest_gpu.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:srht_pass -s 4 -c 2 \
      -o gpurun_out/prof_srht python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_srht.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_srht.log; tail -2 gpurun_out/ncu_srht.log
