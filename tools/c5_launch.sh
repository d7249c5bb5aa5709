cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT; mkdir -p gpurun_out/prof
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof/launches_c5.csv python bench.py --config c5 --rows 1000000 --steps 1 --warmup 2 --no-e2e --no-cpu > /dev/null 2>&1
echo "exit $?"
