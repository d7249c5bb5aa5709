#!/bin/bash
# K1 with the cooperative grouping vs the radix grouping (LVSK_GROUP_RADIX=1)
export PYTHONPATH=$GRAFT_REPO_ROOT
for i in 1 2; do
  python tools/k1_time.py
  LVSK_GROUP_RADIX=1 python tools/k1_time.py
done
