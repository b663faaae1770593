#!/bin/bash
# Builds experiment variants of the library (here, CPU) into paper_2508_14568_b200/_build_<name>/
# usage: tools/variants.sh name1:DEF=V,DEF2=V name2:...   (design tool)
set -e
cd "$(dirname "$0")/.."
for spec in "$@"; do
  name=${spec%%:*}; defs=${spec#*:}
  args=""
  if [ "$defs" != "$name" ]; then for d in ${defs//,/ }; do args="$args $d"; done; fi
  python paper_2508_14568_b200/build.py $args --out paper_2508_14568_b200/_build_$name > /dev/null
  echo "built $name ($args)"
done
