#!/bin/bash
# One gpurun call: GPU tests, bench line, launch list and ncu captures.
mkdir -p gpurun_out
TAG=${TAG:-r1}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15
timeout 600 python bench.py --steps 20 --warmup 5 2>&1 | tail -3 | tee gpurun_out/bench_$TAG.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k 'regex:plx::' -c 400 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/ncu_launch_stdout.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:march_bwd|colour_kernel|scatter_kernel' -s 36 -c 3 -o gpurun_out/prof_render_$TAG python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_full_stdout.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:touched_compact|opt_rows' -s 24 -c 2 -o gpurun_out/prof_opt_$TAG python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/ncu_full_opt_stdout.log 2>&1
ls -la gpurun_out
