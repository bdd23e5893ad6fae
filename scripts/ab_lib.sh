#!/bin/bash
# A/B two in-tree libcf builds on the same box: bash scripts/ab_lib.sh <cmd...>
# (runs the command alternately with libcf_head.so and libcf.so, twice)
for i in 1 2; do
  for v in libcf_head.so libcf.so; do
    echo "== $v"
    CF_LIB_PATH=$PWD/paper_2504_09014_b200/$v "$@"
  done
done
