# round-2 (session 3) profiles: gpu tests, every config's bench line, launch
# lists, full ncu captures of the kernels changed this session (under gpurun)
cd $GRAFT_REPO_ROOT
export PYTHONPATH=$GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof3
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 > gpurun_out/prof3/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/prof3/pytest.log
tail -2 gpurun_out/prof3/pytest.log
for c in c1 c2 c3 c4 c5; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/prof3/bench_$c.log 2>&1
  echo "$c exit $?"; tail -1 gpurun_out/prof3/bench_$c.log | grep -o "\"ms_per_step\": [0-9.]*"
done
for c in c2 c4; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof3/launches_$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
  echo "launches $c exit $?"
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:csr_sketch_kernel -c 1 -o gpurun_out/prof3/k2 python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/prof3/ncu_k2.log 2>&1; echo "k2 $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:chol_fold_kernel -c 1 -o gpurun_out/prof3/kf_c4 python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/prof3/ncu_kf4.log 2>&1; echo "kf4 $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:chol_fold_kernel -c 1 -o gpurun_out/prof3/kf_c2 python bench.py --config c2 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/prof3/ncu_kf2.log 2>&1; echo "kf2 $?"
ls gpurun_out/prof3
