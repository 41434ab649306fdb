#!/bin/bash
# Round-2 profiling evidence (one GPU): ncu --set full of the three render
# kernels + the update at the C2 headline state, and of the render kernels
# at C5 B = 2^18 and 2^20 (L2 hit rate, L2 red sectors, DRAM bytes), plus the
# launch list of the default bench command.
mkdir -p gpurun_out
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
# C2 headline: warm-up 5 steps, then kernels of step 5 (prologue, march, colour, scatter, tv, compact, opt)
timeout 900 $NCU -k "regex:march_bwd|colour_kernel|scatter_kernel|opt_rows|tv_dense_kernel|tv_sparse_kernel" -s 30 -c 5 \
  -o gpurun_out/prof_c2_r2 python bench.py --steps 3 --warmup 5 --no-cpu-baseline --steady-step 0 \
  > gpurun_out/prof_c2_r2.log 2>&1
# C5 at 2^18 (6 waves/step) and 2^20: render kernels of the first wave after 3 warm-up steps
STEPS=1 WARM=3 LOGB0=18 LOGB1=19 timeout 900 $NCU -k "regex:march_bwd|colour_kernel|scatter_kernel" \
  -s 63 -c 3 -o gpurun_out/prof_c5_18_r2 python scripts/sweep_c5.py > gpurun_out/prof_c5_18_r2.log 2>&1
STEPS=1 WARM=2 LOGB0=20 LOGB1=21 timeout 900 $NCU -k "regex:march_bwd|colour_kernel|scatter_kernel" \
  -s 150 -c 3 -o gpurun_out/prof_c5_20_r2 python scripts/sweep_c5.py > gpurun_out/prof_c5_20_r2.log 2>&1
# launch list of the default bench command (per-launch durations, serialised)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_r2.csv python bench.py --steps 3 --warmup 5 --no-cpu-baseline \
  --steady-step 0 > gpurun_out/launches_r2.log 2>&1
ls -la gpurun_out/*.ncu-rep
