set -x
python -c 'import __graft_entry__ as g; g.build()'
export ADAPTRA_TIMEOUT_MS=60000
timeout 600 python bench.py > gpurun_out/r02dd_bench_default.json 2> gpurun_out/r02dd_bench_default.err; echo bench rc=$?
tail -c 600 gpurun_out/r02dd_bench_default.json
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/r02dd_smoke.txt 2>&1; echo smoke rc=$?
timeout 2700 python -m pytest tests -m gpu -x -q > gpurun_out/r02dd_pytest_gpu.txt 2>&1; echo all rc=$?
tail -3 gpurun_out/r02dd_pytest_gpu.txt
