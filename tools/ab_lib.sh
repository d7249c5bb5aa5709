#!/bin/bash
# A/B two builds of the native library on one command: ab_lib.sh <libA> <libB> <cmd...>
A=$1; B=$2; shift 2
cp paper_1812_07903_b200/liblevsketch_b200.so /tmp/lib_cur.so
for L in $A $B $A $B; do cp $L paper_1812_07903_b200/liblevsketch_b200.so; echo "== $L"; "$@"; done
cp /tmp/lib_cur.so paper_1812_07903_b200/liblevsketch_b200.so
