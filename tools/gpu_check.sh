cd $GRAFT_REPO_ROOT
export PYTHONPATH=$GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 > gpurun_out/pytest_all.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_all.log
tail -12 gpurun_out/pytest_all.log
timeout 300 python tools/kf_time.py > gpurun_out/kf_time.log 2>&1; cat gpurun_out/kf_time.log
timeout 300 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu > gpurun_out/bench_c2.log 2>&1
echo "bench c2 exit $?" >> gpurun_out/bench_c2.log; tail -c 1300 gpurun_out/bench_c2.log
timeout 300 python bench.py --config c5 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_c5.log 2>&1
echo "bench c5 exit $?" >> gpurun_out/bench_c5.log; tail -c 1300 gpurun_out/bench_c5.log
