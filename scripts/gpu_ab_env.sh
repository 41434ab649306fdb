#!/bin/bash
# A/B of an environment switch: kernel times and bench value under each setting.
# usage: VAR=PLX_PREFETCH VALUES="0 1" bash scripts/gpu_ab_env.sh
for v in $VALUES; do
  echo "== $VAR=$v"
  env $VAR=$v python scripts/kernel_times.py 20 5 2>/dev/null | head -4
  env $VAR=$v python scripts/kernel_times.py 20 2000 2>/dev/null | head -2
done
