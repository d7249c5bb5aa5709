cd $GRAFT_REPO_ROOT; export PYTHONPATH=$GRAFT_REPO_ROOT
bash tools/ab_lib.sh ab/old.so ab/new.so bash -c 'timeout 300 python tools/kf_time.py 2>&1 | grep -o "kf_us.: [0-9.]*" | tr "\n" " "; echo; timeout 300 python bench.py --config c2 --steps 30 --warmup 5 --no-e2e --no-cpu 2>&1 | tail -1 | grep -o "\"ms_per_step\": [0-9.]*\|\"factor_ms\": [0-9.]*" | tr "\n" " "; echo'
