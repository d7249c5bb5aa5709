# round-2 profiles: launch lists + full ncu captures (run under gpurun)
cd $GRAFT_REPO_ROOT
export PYTHONPATH=$GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof2
for c in c2 c4 c5; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof2/launches_$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
  echo "launches $c exit $?"
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:csr_sketch_kernel -c 1 -o gpurun_out/prof2/k2 python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/prof2/ncu_k2.log 2>&1; echo "k2 $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:csr_rowsumsq -c 1 -o gpurun_out/prof2/k6 python bench.py --config c4 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/prof2/ncu_k6.log 2>&1; echo "k6 $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gaussian_tc_pair_kernel -c 1 -o gpurun_out/prof2/k4pair python bench.py --config c5 --rows 1000000 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/prof2/ncu_k4.log 2>&1; echo "k4 $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:leverage_bf16_pair -c 1 -o gpurun_out/prof2/k5bf16 python bench.py --config c5 --rows 1000000 --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/prof2/ncu_k5b.log 2>&1; echo "k5b $?"
ls -la gpurun_out/prof2
