# session-3 late captures: C2 launch list with KD, ncu of KD (syrk) and KM (merge)
cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT; mkdir -p gpurun_out/prof4
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/prof4/launches_c2.csv python bench.py --config c2 --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1; echo "launches $?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:syrk_kernel -c 1 -o gpurun_out/prof4/kd python bench.py --config c2 --steps 1 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1; echo "kd $?"
timeout 600 ncu --set full --clock-control none -k regex:km_merge_kernel -c 3 -o gpurun_out/prof4/km python tools/merge_prof_case.py > /dev/null 2>&1; echo "km $?"
