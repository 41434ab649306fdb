#!/bin/bash
# A/B of the bench headline and steady-state lines under an environment
# switch: scripts/bench_ab_env.sh "PLX_X=1" [rounds]
ENV_B="$1"; N="${2:-2}"
pick='import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d["value"], d["ms_per_step"], d["config"]["steady_state"]["rays_per_s"], d["e2e"]["value"])'
for i in $(seq "$N"); do
  echo "A $(python bench.py 2>/dev/null | python -c "$pick")"
  echo "B $(env $ENV_B python bench.py 2>/dev/null | python -c "$pick")"
done
