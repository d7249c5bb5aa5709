# every config's bench line (run under gpurun)
cd $GRAFT_REPO_ROOT
export PYTHONPATH=$GRAFT_REPO_ROOT
mkdir -p gpurun_out/bench_r2
for c in c1 c2 c3 c4 c5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu > gpurun_out/bench_r2/bench_$c.log 2>&1
  echo "$c exit $?"; tail -1 gpurun_out/bench_r2/bench_$c.log | grep -o '"ms_per_step": [0-9.]*\|"stages_ms": {[^}]*}[^}]*}[^}]*}\|"e2e": {"value": [0-9.e+]*'
done
