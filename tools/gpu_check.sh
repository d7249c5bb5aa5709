cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 -k "srht or fwht or explicit" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config c3 --steps 30 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_c3.log 2>&1
echo "bench c3 exit $?" >> gpurun_out/bench_c3.log; tail -2 gpurun_out/bench_c3.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv \
      python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch_c3.log 2>&1
