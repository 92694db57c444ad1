set -x
python -c 'import __graft_entry__ as g; g.build()'
timeout 900 python -m pytest tests/test_gpu_stage.py tests/test_gpu_fullsize.py tests/test_gpu_pipeline.py -x -q > gpurun_out/r02_pytest_gpu_5a.txt 2>&1; echo pytest_a rc=$?
tail -3 gpurun_out/r02_pytest_gpu_5a.txt
timeout 1200 python bench.py --arms adaptive,zb --no-cpu > gpurun_out/r02_bench_5.json 2> gpurun_out/r02_bench_5.err; echo bench rc=$?
ADAPTRA_W_PAIRS=0 timeout 1200 python bench.py --arms adaptive --no-e2e --no-cpu > gpurun_out/r02_bench_5_nopairs.json 2> gpurun_out/r02_bench_5_nopairs.err; echo bench rc=$?
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02_pytest_gpu_5.txt 2>&1; echo pytest rc=$?
tail -3 gpurun_out/r02_pytest_gpu_5.txt
