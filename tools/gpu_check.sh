cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -25 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --config c5 --steps 3 --warmup 1 --no-e2e --no-cpu > gpurun_out/bench_c5.log 2>&1
echo "bench c5 exit $?" >> gpurun_out/bench_c5.log; tail -3 gpurun_out/bench_c5.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv \
      python bench.py --config c5 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch_c5.log 2>&1
