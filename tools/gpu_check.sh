cd $GRAFT_REPO_ROOT
export PYTHONPATH=$GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 -k "cholesky or pipeline_fold or gaussian or c5 or jl_fold" > gpurun_out/pytest_sel.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_sel.log
tail -12 gpurun_out/pytest_sel.log
timeout 300 python bench.py --config c5 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_c5.log 2>&1
echo "bench c5 exit $?" >> gpurun_out/bench_c5.log; tail -c 1300 gpurun_out/bench_c5.log
timeout 300 python bench.py --config c1 --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_c1.log 2>&1
echo "bench c1 exit $?" >> gpurun_out/bench_c1.log; tail -c 1300 gpurun_out/bench_c1.log
