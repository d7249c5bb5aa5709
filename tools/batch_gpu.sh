# BatchRunner parity + pipelined bench lines
cd $GRAFT_REPO_ROOT
export PYTHONPATH=$GRAFT_REPO_ROOT
mkdir -p gpurun_out/batch
timeout 600 python -m pytest tests/test_gpu_batch.py -q --timeout 300 2>&1 | tail -3
for c in c2 c1 c3; do
  timeout 400 python bench.py --config $c --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/batch/bench_$c.log 2>&1; echo "$c exit $?"
  tail -1 gpurun_out/batch/bench_$c.log | python -c "import json,sys; b=json.loads(sys.stdin.read()); print(b['config'].get('workload'), b['ms_per_step'], b.get('latency_ms_per_pass'), b['roofline']['frac'], b['stages_ms'])"
done
timeout 400 python bench.py --config c2 --steps 20 --warmup 3 --no-e2e --no-cpu --inflight 1 2>&1 | tail -1 | cut -c1-200
