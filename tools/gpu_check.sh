cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python tools/tc_smoke.py > gpurun_out/tc_smoke.log 2>&1; echo "tc_smoke exit $?" >> gpurun_out/tc_smoke.log
cat gpurun_out/tc_smoke.log
grep -q "tc_smoke exit 0" gpurun_out/tc_smoke.log || exit 1
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 200 --warmup 5 --e2e-steps 3 --cpu-rows 100000 > gpurun_out/bench.log 2>&1
echo "bench exit $?" >> gpurun_out/bench.log
tail -2 gpurun_out/bench.log
for c in c3 c1; do
  timeout 600 python bench.py --config $c --steps 30 --warmup 3 --no-e2e --cpu-rows 20000 > gpurun_out/bench_$c.log 2>&1
  echo "bench $c exit $?" >> gpurun_out/bench_$c.log; tail -2 gpurun_out/bench_$c.log
done
if grep -q "bench exit 0" gpurun_out/bench.log; then
  timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:hashed_gather -s 1 -c 1 \
      -o gpurun_out/prof_gather python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_gather.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:leverage_v2 -s 1 -c 1 \
      -o gpurun_out/prof_k5 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_k5.log 2>&1
  echo "ncu exit $?" >> gpurun_out/ncu_launch.log
fi
