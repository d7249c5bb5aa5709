# Round profile capture: tests, every config's bench line, launch lists and
# full ncu sets of the kernels changed this round (run under gpurun).
cd $GRAFT_REPO_ROOT
export PYTHONPATH=$GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 > gpurun_out/prof/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/prof/pytest.log
tail -2 gpurun_out/prof/pytest.log
for c in c1 c2 c3 c4 c5; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/prof/bench_$c.log 2>&1
  echo "$c exit $?"; tail -1 gpurun_out/prof/bench_$c.log | grep -o "\"ms_per_step\": [0-9.]*"
done
for c in c1 c3 c4 c5; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_$c.csv python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:srht_sampled_kernel -c 1 -o gpurun_out/prof/k3 python bench.py --config c3 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gaussian_tc_kernel -c 1 -o gpurun_out/prof/k4 python bench.py --config c5 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:csr_stream -c 1 -o gpurun_out/prof/k2 python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
ls gpurun_out/prof
