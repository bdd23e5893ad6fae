#!/bin/bash
# Build libcf variants on the box (EXTRA defines) and A/B them against libcf.so:
#   bash scripts/ab_builds.sh "name1:-DFOO" "name2:-DBAR -DBAZ" -- <cmd...>
cd "$(dirname "$0")/.."
variants=()
while [ "$1" != "--" ]; do variants+=("$1"); shift; done
shift
for v in "${variants[@]}"; do
  name=${v%%:*}; flags=${v#*:}
  make -s -C paper_2504_09014_b200/csrc EXTRA="$flags" OUT=../libcf_$name.so OBJDIR=/tmp/obj_$name -j16 >/dev/null 2>&1 || echo "build $name failed"
done
for i in 1 2; do
  echo "== base"; "$@"
  for v in "${variants[@]}"; do
    name=${v%%:*}; echo "== $name"; CF_LIB_PATH=$PWD/paper_2504_09014_b200/libcf_$name.so "$@"
  done
done
