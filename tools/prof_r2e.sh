# session-5: every GPU test, C4 bench after K6-TC v2, C4 launch list, ncu of K6-TC v2
cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT; mkdir -p gpurun_out/prof5
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 > gpurun_out/prof5/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/prof5/pytest.log
tail -2 gpurun_out/prof5/pytest.log
timeout 600 python bench.py --config c4 --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/prof5/bench_c4.log 2>&1; echo "c4 exit $?"
timeout 600 python tools/k6v2_time.py 4000000 10 > gpurun_out/prof5/k6v2_time.log 2>&1; tail -2 gpurun_out/prof5/k6v2_time.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof5/launches_c4.csv python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu --inflight 1 > /dev/null 2>&1; echo "launches $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:csr_rowsumsq_tc2_kernel -c 1 -o gpurun_out/prof5/k6v2 python bench.py --config c4 --steps 1 --warmup 1 --no-e2e --no-cpu --inflight 1 > /dev/null 2>&1; echo "k6v2 ncu $?"
