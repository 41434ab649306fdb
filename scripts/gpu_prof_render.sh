#!/bin/bash
# Source-level ncu capture of the three render-backward kernels at the C2
# headline state (step 5 after the dense init) -> gpurun_out/prof_render_$TAG.ncu-rep
mkdir -p gpurun_out
TAG=${TAG:-a}
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 900 $NCU -k "regex:march_bwd|colour_kernel|scatter_kernel" -s 18 -c 3 \
  -o gpurun_out/prof_render_$TAG python bench.py --steps 3 --warmup 5 --no-cpu-baseline --steady-step 0 \
  > gpurun_out/prof_render_$TAG.log 2>&1
ls -la gpurun_out/
