#!/bin/bash
# Per-kernel CUPTI times (scripts/kernel_times.py) of library variants / diag modes:
#   RUNS="base diag:1 diag:6" -> libplx.so, libplx_diag.so with PLX_DIAG_MODE=1, =6
mkdir -p gpurun_out
for r in ${RUNS:-base}; do
  v=${r%%:*}; m=${r#*:}; [ "$m" = "$r" ] && m=0
  if [ "$v" = base ]; then L=""; else L="PLX_LIB=$PWD/paper_2112_05131_b200/libplx_$v.so"; fi
  echo "== $r"
  env $L PLX_TV_SERIAL=1 PLX_DIAG_MODE=$m timeout 300 python scripts/kernel_times.py 20 ${WARM:-5} 2>&1 | grep -E "us/step|device-timed" | head -16
done > gpurun_out/diag_${TAG:-a}.txt 2>&1
cat gpurun_out/diag_${TAG:-a}.txt
