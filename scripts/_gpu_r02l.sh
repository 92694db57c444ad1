set -x
python -c 'import __graft_entry__ as g; g.build()'
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_stage.py tests/test_gpu_toggles.py -x -q > gpurun_out/r02_pytest_gpu_8a.txt 2>&1; echo pa rc=$?
tail -3 gpurun_out/r02_pytest_gpu_8a.txt
timeout 1200 python bench.py --replan-log gpurun_out/r02_replan_log_c3_s8_1gpu_b8.jsonl > gpurun_out/r02_bench_8.json 2> gpurun_out/r02_bench_8.err; echo bench rc=$?
tail -2 gpurun_out/r02_bench_8.err
