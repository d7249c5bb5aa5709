cd $GRAFT_REPO_ROOT
export PYTHONPATH=$GRAFT_REPO_ROOT
mkdir -p gpurun_out
LVSK_KF_TRACE=1 timeout 300 python tools/kf_time.py > gpurun_out/kf_trace.log 2>&1; grep -m 8 "KF d=\|kf_us" gpurun_out/kf_trace.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gaussian_tc_kernel -c 1 -o gpurun_out/prof_gauss_tc -f python bench.py --config c5 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_gauss.log 2>&1; tail -3 gpurun_out/ncu_gauss.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:chol_fold -c 1 -o gpurun_out/prof_kf -f python tools/kf_time.py > gpurun_out/ncu_kf.log 2>&1; tail -2 gpurun_out/ncu_kf.log
