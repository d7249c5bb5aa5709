# fp32 Gaussian: stacked-plane K4-TC parity + error probe + C1 bench line + launch list
cd $GRAFT_REPO_ROOT
export PYTHONPATH=$GRAFT_REPO_ROOT
mkdir -p gpurun_out/k4f32
timeout 300 python tools/k4f32_err.py
timeout 600 python -m pytest tests -m gpu -q -k "gaussian or config" --timeout 300 2>&1 | tail -3
for i in 1 2; do timeout 300 python bench.py --config c1 --steps 20 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | cut -c1-300; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/k4f32/launches_c1.csv \
  python bench.py --config c1 --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1; echo "ncu exit $?"
