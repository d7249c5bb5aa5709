cd $GRAFT_REPO_ROOT
export PYTHONPATH=$GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -rf --timeout 300 -k "gaussian or c5" > gpurun_out/pytest_g.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_g.log
tail -8 gpurun_out/pytest_g.log
timeout 300 python tools/kf_time.py > gpurun_out/kf_time.log 2>&1; cat gpurun_out/kf_time.log
timeout 300 python bench.py --config c5 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_c5.log 2>&1
echo "bench c5 exit $?" >> gpurun_out/bench_c5.log; tail -c 1500 gpurun_out/bench_c5.log
timeout 300 ncu --metrics gpu__time_duration.sum,sm__inst_executed.sum,smsp__cycles_active.avg --clock-control none -k regex:chol_fold -c 3 python tools/kf_time.py > gpurun_out/kf_ncu.log 2>&1; grep -E "chol_fold|duration|inst_exec|cycles_active" gpurun_out/kf_ncu.log | head -20
