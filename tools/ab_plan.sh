#!/bin/bash
# A/B of the plan variants on the bench workloads (development): cluster size and tail fusion.
for cl in 1 8; do
  for fuse in 1 0; do
    echo "== STAR_PLAN_CLUSTER=$cl STAR_PLAN_FUSE=$fuse"
    STAR_PLAN_CLUSTER=$cl STAR_PLAN_FUSE=$fuse python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline --no-sweep "$@" \
      | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['config']['workload'][:4], 'us', round(d['us_per_step'],2), 'warm', d['step_us_warm_l2'], 'stage', d['stage_us'].get('plan'), 'moves', d['plan_stats'])"
  done
done
