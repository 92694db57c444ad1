set -x
python -c 'import __graft_entry__ as g; g.build()'
timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_stage.py -x -q > gpurun_out/r02_pytest_gpu_4a.txt 2>&1; echo pytest_a rc=$?
tail -3 gpurun_out/r02_pytest_gpu_4a.txt
REPS=20 timeout 300 python scripts/gemm_bench.py > gpurun_out/r02_gemm_bn128.jsonl 2>&1; echo rc=$?
ADAPTRA_GEMM_BN=256 REPS=20 timeout 300 python scripts/gemm_bench.py > gpurun_out/r02_gemm_bn256.jsonl 2>&1; echo rc=$?
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02_pytest_gpu_4.txt 2>&1; echo pytest rc=$?
tail -3 gpurun_out/r02_pytest_gpu_4.txt
timeout 1200 python bench.py --arms adaptive,zb > gpurun_out/r02_bench_4.json 2> gpurun_out/r02_bench_4.err; echo bench rc=$?
ADAPTRA_GEMM_BN=256 ADAPTRA_W_PAIRS=0 timeout 1200 python bench.py --arms adaptive --no-e2e --no-cpu > gpurun_out/r02_bench_4_old.json 2> gpurun_out/r02_bench_4_old.err; echo bench rc=$?
