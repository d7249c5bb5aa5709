cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -30 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 50 --warmup 3 --e2e-steps 3 --cpu-rows 100000 > gpurun_out/bench.log 2>&1
echo "bench exit $?" >> gpurun_out/bench.log
tail -3 gpurun_out/bench.log
if grep -q "bench exit 0" gpurun_out/bench.log; then
  timeout 600 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:hashed_gather -s 1 -c 1 \
      -o gpurun_out/prof_gather python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_gather.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:leverage_tf32x3 -s 1 -c 1 \
      -o gpurun_out/prof_k5 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_k5.log 2>&1
  echo "ncu exit $?" >> gpurun_out/ncu_launch.log
fi
