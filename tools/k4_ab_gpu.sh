cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
cp paper_1812_07903_b200/liblevsketch_b200.so /tmp/lib_cur.so
cp ab/new.so paper_1812_07903_b200/liblevsketch_b200.so
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -k "gaussian or c1 or c5" --timeout 300 2>&1 | tail -3
for L in ab/old.so ab/new.so ab/old.so ab/new.so; do cp $L paper_1812_07903_b200/liblevsketch_b200.so; echo "== $L"; timeout 300 python tools/k4_time.py 2>&1 | tail -4; done
cp ab/new.so paper_1812_07903_b200/liblevsketch_b200.so
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | grep -o '"ms_per_step": [0-9.]*\|"sketch": {"ms": [0-9.]*\|"sm_mhz": [0-9.]*'
cp /tmp/lib_cur.so paper_1812_07903_b200/liblevsketch_b200.so
