# session-5 closing launch list of the default bench command (C2), one pass at a time
cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT; mkdir -p gpurun_out/prof6
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof6/launches_c2.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --inflight 1 > /dev/null 2>&1; echo "launches $?"
