#!/bin/bash
# On the GPU box: BR time of blind-rotation forms/variants: entries name[:form]
cd "$(dirname "$0")/.."
for spec in "$@"; do
  name=${spec%%:*}; form=${spec#*:}; [ "$form" = "$spec" ] && form=""
  if [ "$name" = base ]; then lib=paper_2508_14568_b200/_build/libleuven_b200.so; else lib=paper_2508_14568_b200/_build_$name/libleuven_b200.so; fi
  echo "== $spec: $(LVB_BR_FORM=$form LVB_LIB=$lib timeout 300 python tools/profile_pbs.py 4096 2>&1 | tail -1)"
done
