#!/bin/bash
# On the GPU box: BR/KS time of each built variant on the cfg2 batch.
# usage: tools/run_variants.sh name1 name2 ...   (design tool)
cd "$(dirname "$0")/.."
for name in "$@"; do
  if [ "$name" = base ]; then lib=paper_2508_14568_b200/_build/libleuven_b200.so; else lib=paper_2508_14568_b200/_build_$name/libleuven_b200.so; fi
  echo "== $name: $(LVB_LIB=$lib timeout 300 python tools/profile_pbs.py 4096 2>&1 | tail -1)"
done
