#!/bin/bash
# A/B several in-tree libcf builds on the same box, alternating, twice:
# LIBS="libcf_head.so libcf.so ..." bash scripts/ab_libs.sh <cmd...>
for i in 1 2; do
  for v in ${LIBS:-libcf_head.so libcf.so}; do
    echo "== $v"
    CF_LIB_PATH=$PWD/paper_2504_09014_b200/$v "$@"
  done
done
