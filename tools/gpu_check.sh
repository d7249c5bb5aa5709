cd $GRAFT_REPO_ROOT
export PYTHONPATH=$GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_c4.log 2>&1
echo "bench c4 exit $?" >> gpurun_out/bench_c4.log; tail -c 1500 gpurun_out/bench_c4.log
LVSK_K2_SIMPLE=1 timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_c4_simple.log 2>&1
echo "bench c4 simple exit $?" >> gpurun_out/bench_c4_simple.log; tail -c 700 gpurun_out/bench_c4_simple.log
timeout 300 python bench.py --config c3 --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_c3.log 2>&1
echo "bench c3 exit $?" >> gpurun_out/bench_c3.log; tail -c 1200 gpurun_out/bench_c3.log
timeout 600 python bench.py > gpurun_out/bench_default.log 2>&1
echo "bench default exit $?" >> gpurun_out/bench_default.log; tail -c 2500 gpurun_out/bench_default.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch_c2.log 2>&1; tail -2 gpurun_out/ncu_launch_c2.log
