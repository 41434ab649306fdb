timeout 2400 python -m pytest tests -q -m gpu --timeout 1200 2>&1 | tail -3
bash scripts/ab_bench.sh cur ""
C3_PROFILE=1 timeout 900 python scripts/ladder_c3.py 2>/dev/null | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('C3', d['ms_per_step_256'], d['rays_per_s_256'], d['ms_per_step_512'], d['rays_per_s_512'], d['rung_event_ms_device']); print(json.dumps(d['kernel_us_per_step_512']))"
