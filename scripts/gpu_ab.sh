#!/bin/bash
# A/B of kernel variants: parity under each, then bench lines.
mkdir -p gpurun_out
TAG=${TAG:-ab}
PLX_BWD_MINB=3 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
for v in 2 3; do
  PLX_BWD_MINB=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_${TAG}_minb$v.json
  python -c "import json;d=json.load(open('gpurun_out/bench_${TAG}_minb$v.json'));print('minb',$v,d['value'],d['e2e']['value'],d['config']['kernel_ms'],d['clocks'])"
done
