# KF with segmented UPD/WUPD tasks: parity tests, timing, C4/C2 bench
cd $GRAFT_REPO_ROOT
export PYTHONPATH=$GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py -q -x -k "chol or kf or jl or fold or cert or batch or exact or rank" --timeout 300 2>&1 | tail -2
timeout 300 python tools/kf_big_trace.py 2>&1 | grep "KF [0-9]"
timeout 300 python tools/kf_c1_probe.py 2>&1 | grep "KF [0-9]"
for c in c4 c2; do timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | python -c "import json,sys; b=json.loads(sys.stdin.read()); print('$c', b['ms_per_step'], b.get('latency_ms_per_pass'), b['stages_ms']['factor_ms'])"; done
