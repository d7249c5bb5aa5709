# round-2 closing check: every GPU test, smoke, every config's bench line, the default bench + reference arm
cd $GRAFT_REPO_ROOT
export PYTHONPATH=$GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 > gpurun_out/final/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/final/pytest.log
tail -2 gpurun_out/final/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for c in c1 c3 c4 c5; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/final/bench_$c.log 2>&1
  echo "$c exit $?"
done
timeout 900 python bench.py > gpurun_out/final/bench_c2.log 2>&1; echo "c2 default exit $?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final/bench_ref.log 2>&1; echo "ref exit $?"
