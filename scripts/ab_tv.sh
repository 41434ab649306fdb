pick='import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d["value"], d["ms_per_step"], d["config"]["steady_state"]["rays_per_s"], d["e2e"]["value"])'
for i in 1 2; do
for cfg in "PLX_NONE=1" "PLX_PRIO=1" "PLX_PRIO=1 PLX_TV_SHORT=1" "PLX_TV_SHORT=1"; do
  echo "$cfg $(env $cfg python bench.py 2>/dev/null | python -c "$pick")"
done; done
PLX_PRIO=1 PLX_TV_SHORT=1 KT_TIMELINE=1 python scripts/kernel_times.py 20 5 2>/dev/null | head -8
