cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
cp paper_1812_07903_b200/liblevsketch_b200.so /tmp/lib_cur.so
for L in ab/a.so ab/b.so ab/c.so ab/a.so ab/b.so; do cp $L paper_1812_07903_b200/liblevsketch_b200.so; echo "== $L"; timeout 300 python tools/k6v2_time.py 4000000 8 10 12 2>&1 | grep -o "'hot_blocks': [0-9]*, 'ms': [0-9.]*" | tr "\n" ";"; echo; done
cp /tmp/lib_cur.so paper_1812_07903_b200/liblevsketch_b200.so
