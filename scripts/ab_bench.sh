#!/bin/bash
# A/B of library variants / env switches on the C2 bench (no CPU leg):
#   scripts/ab_bench.sh TAG "ENV=.. ENV2=.." [TAG2 "ENV.."] ...
# Each variant runs the bench twice; prints value, steady-state and per-leg ms.
mkdir -p gpurun_out
while [ $# -gt 0 ]; do
  TAG=$1; ENVS=$2; shift 2
  for rep in 1 2; do
    env $ENVS timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ab_$TAG.$rep.json 2> gpurun_out/ab_$TAG.$rep.err
    python - "$TAG" "gpurun_out/ab_$TAG.$rep.json" <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    st = d.get("stats") or d.get("config")
    print(f"{sys.argv[1]:>12}  value {d['value']/1e6:6.3f} M  e2e {d['e2e']['value']/1e6:6.3f} M  "
          f"step2000 {st['steady_state']['rays_per_s']/1e6:6.2f} M  legs " +
          " ".join(f"{k}={v*1000:.1f}us" for k, v in st['kernel_ms'].items()))
except Exception as e:
    print(sys.argv[1], "FAILED", e, open(sys.argv[2].replace('.json', '.err')).read()[-800:])
PY
  done
done
