# compute-sanitizer memcheck / racecheck / synccheck over a -m gpu subset covering
# K1, K2, K3, K4-TC, K5, K6, KF and K7 (run under gpurun; small shapes)
cd $GRAFT_REPO_ROOT
export PYTHONPATH=$GRAFT_REPO_ROOT
mkdir -p gpurun_out/san
SEL="hashed_sketch_bit_exact_f32_and_bf16 or srht_matches_reference or gaussian_tc_bf16_vs_oracle or tcgen05_leverage_vs_fp64 or kf_cholesky_fold_kernel_vs_numpy or argsort_matches_numpy_stable or csr_sketch_bit_exact_vs_dense or csr_leverage_vs_oracle or tcgen05_bf16_leverage_vs_fp64 or gaussian_entries_bit_exact or order_golden"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --target-processes all --print-limit 20 --error-exitcode 99 \
    python -m pytest tests/test_gpu_parity.py -q -x -k "$SEL" -p no:cacheprovider > gpurun_out/san/$tool.log 2>&1
  echo "$tool exit $?"; tail -4 gpurun_out/san/$tool.log
done
