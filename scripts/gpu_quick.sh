#!/bin/bash
# Quick iteration: parity tests, bench line, optional ncu capture of the render / opt kernels.
mkdir -p gpurun_out
TAG=${TAG:-q}
timeout 600 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} 2>&1 | tail -15
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | tee gpurun_out/bench_$TAG.json
if [ -n "$NCU" ]; then
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:march_bwd|colour_kernel|scatter_kernel' -s 36 -c 3 -o gpurun_out/prof_render_$TAG python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_full_stdout.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:touched_compact|opt_rows' -s 24 -c 2 -o gpurun_out/prof_opt_$TAG python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_full_opt_stdout.log 2>&1
fi
