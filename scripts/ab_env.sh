#!/bin/bash
# development A/B: scripts/ab_env.sh "<bench args>" "ENV=.. ENV=.." "ENV=.." ...
args=$1; shift
for envs in "$@"; do
  r=$(env $envs timeout 200 python bench.py $args --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()}, d['count'])" 2>&1)
  echo "[$args] [$envs] $r"
done
