mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/gputests_v1.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputests_v1.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_v1.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_v1.json 2> gpurun_out/bench_v1.err
