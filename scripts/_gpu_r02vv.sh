set -x
python -c 'import __graft_entry__ as g; g.build()'
export ADAPTRA_TIMEOUT_MS=60000
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/r02vv_smoke.txt 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests/test_gpu_stage.py tests/test_gpu_fullsize.py tests/test_gpu_pipeline.py -x -q > gpurun_out/r02vv_pytest.txt 2>&1; echo st rc=$?
tail -1 gpurun_out/r02vv_pytest.txt
timeout 300 python bench.py > gpurun_out/r02vv_bench_default.json 2> gpurun_out/r02vv_bench_default.err; echo bench rc=$?
