#!/bin/bash
# A/B of kernel variants: parity under each, then bench lines.
mkdir -p gpurun_out
TAG=${TAG:-ab}
VARIANTS=${VARIANTS:-"4 5 6"}
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for v in $VARIANTS; do
  PLX_BWD_MINB=$v timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k backward 2>&1 | tail -1
  PLX_BWD_MINB=$v timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_${TAG}_minb$v.json
  python -c "import json;d=json.load(open('gpurun_out/bench_${TAG}_minb$v.json'));c=d['config'];print('minb',$v,round(d['value']),round(d['e2e']['value']),c['kernel_ms'],c['march_positions_per_step'],c['samples_per_step'],c['chunks_per_step'])"
done
