# K4-TC profile + config parity tests (run under gpurun)
cd $GRAFT_REPO_ROOT
export PYTHONPATH=$GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof
timeout 1200 python -m pytest tests/test_gpu_configs.py -q -rf -s --timeout 900 > gpurun_out/prof/pytest_configs.log 2>&1; echo "pytest exit $?" >> gpurun_out/prof/pytest_configs.log
tail -3 gpurun_out/prof/pytest_configs.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gaussian_tc_kernel -c 1 -o gpurun_out/prof/k4 python bench.py --config c5 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/prof/ncu_k4.log 2>&1
echo "ncu exit $?"
ls gpurun_out/prof
