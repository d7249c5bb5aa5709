cd $GRAFT_REPO_ROOT
export PYTHONPATH=$GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 > gpurun_out/pytest_all.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_all.log
tail -6 gpurun_out/pytest_all.log
for c in c1 c2 c3 c4 c5; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_$c.log 2>&1
  echo "$c exit $?"; grep -o "\"ms_per_step\": [0-9.]*\|\"stages_ms\": {[^}]*}[^}]*}[^}]*}" gpurun_out/bench_$c.log
done
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
