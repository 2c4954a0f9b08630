#!/bin/bash
# development: enum/prep times of C4, C3 (6,3), C3 (3,6), C2 and C5 (one GPU)
for a in "C4" "C3 --p 6 --q 3" "C3 --p 3 --q 6" "C2"; do
  timeout 200 python bench.py --config $a --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['config']['workload'], round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()}, d['count'])"
done
BC_DEBUG=1 REPS=2 timeout 300 python scripts/c5_probe.py 8 8 2>&1 | grep -v "bc prep"
