#!/bin/bash
# Round-2 closing evidence in one gpurun call: GPU suite, smoke, the
# driver-equivalent bench lines (ours + reference arm), the launch list of
# the bench command, warm-cache per-kernel DRAM traffic of the timed steps,
# ncu --set full of the render and update kernels, the C5 sweep and the 360 line.
mkdir -p gpurun_out
TAG=${TAG:-r2c}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi_$TAG.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 > gpurun_out/gputest_$TAG.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
NB="python bench.py --steps 3 --warmup 5 --no-cpu-baseline --steady-step 0"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_$TAG.csv $NB > /dev/null 2>&1
# warm-cache traffic over the same 20-step window bench.py's algorithmic bytes average over
timeout 1200 ncu --cache-control none --clock-control none --kernel-name-base demangled \
  --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
  --log-file gpurun_out/warm_$TAG.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline \
  --steady-step 0 > /dev/null 2>&1
NCU="ncu --set full --clock-control none --import-source on --kernel-name-base demangled"
timeout 900 $NCU -k "regex:march_bwd|colour_kernel|scatter_kernel|opt_rows|tv_dense_kernel|tv_sparse_kernel|touched_compact" -s 36 -c 6 \
  -o gpurun_out/prof_c2_$TAG $NB > /dev/null 2>&1
STEPS=10 WARM=3 timeout 900 python scripts/sweep_c5.py > gpurun_out/sweep_c5_$TAG.log 2>&1
# C5 2^20: the render kernels of one wave (dead-brick mask, spatial segment order)
STEPS=1 WARM=2 LOGB0=20 LOGB1=21 timeout 1200 $NCU -k "regex:march_bwd|colour_kernel|scatter_kernel|seg_" \
  -s 36 -c 6 -o gpurun_out/prof_c5_$TAG python scripts/sweep_c5.py > /dev/null 2>&1
timeout 600 python scripts/bench_msi.py > gpurun_out/msi_$TAG.json 2>&1
timeout 900 python scripts/ladder_c3.py > gpurun_out/c3_$TAG.json 2>/dev/null
timeout 900 python scripts/bench_c4.py > gpurun_out/c4_$TAG.json 2>/dev/null
ls -la gpurun_out
