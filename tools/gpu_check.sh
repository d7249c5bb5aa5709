cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 -k "kf_ or cholesky or csr or jl_fold or leverage_golden or c2_full or distributed or c5" > gpurun_out/pytest_new.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_new.log
tail -15 gpurun_out/pytest_new.log
timeout 300 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu > gpurun_out/bench_c2.log 2>&1
echo "bench c2 exit $?" >> gpurun_out/bench_c2.log; tail -c 1200 gpurun_out/bench_c2.log
timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_c4.log 2>&1
echo "bench c4 exit $?" >> gpurun_out/bench_c4.log; tail -c 1200 gpurun_out/bench_c4.log
timeout 300 python tools/factor_bench.py > gpurun_out/factor_bench.log 2>&1; cat gpurun_out/factor_bench.log
