# every config's bench line (pipelined N=1 default) + the default C2 line with e2e and the CPU baseline
cd $GRAFT_REPO_ROOT
export PYTHONPATH=$GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2d
for c in c1 c3 c4 c5; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/r2d/bench_$c.log 2>&1
  echo "$c exit $?"
done
timeout 900 python bench.py > gpurun_out/r2d/bench_c2.log 2>&1; echo "c2 default exit $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2d/launches_c1.csv python bench.py --config c1 --steps 1 --warmup 3 --no-e2e --no-cpu --inflight 1 > /dev/null 2>&1; echo "launches c1 $?"
