#!/bin/bash
# usage: scripts/ab_test.sh "label:libsuffix:ENV=VAL ..." ...   (runs C2, C3(6,3), C4 per variant)
for spec in "$@"; do
  IFS=: read -r label suf envs <<< "$spec"
  if [ -n "$suf" ]; then export BC_LIB=$GRAFT_REPO_ROOT/paper_2403_07858_b200/libbicount_b200_$suf.so; else unset BC_LIB; fi
  for kv in $envs; do export "$kv"; done
  echo "== $label"
  timeout 100 python scripts/one_count.py C2 4 | tail -2
  timeout 100 python scripts/one_count.py C3 3 6 3 | tail -1
  timeout 100 python scripts/one_count.py C4 3 | tail -1
  for kv in $envs; do unset "${kv%%=*}"; done
done
