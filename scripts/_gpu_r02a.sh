set -x
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv
python -c 'import __graft_entry__ as g; g.build()'
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_pytest_gpu_1.txt 2>&1; echo pytest rc=$?
tail -5 gpurun_out/r02_pytest_gpu_1.txt
timeout 900 python bench.py --steps 8 --warmup 3 --replan-log gpurun_out/r02_replan_log_c1_1gpu.jsonl > gpurun_out/r02_bench_1.json 2> gpurun_out/r02_bench_1.err; echo bench rc=$?
tail -3 gpurun_out/r02_bench_1.err
