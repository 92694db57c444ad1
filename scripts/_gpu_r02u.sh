set -x
python -c 'import __graft_entry__ as g; g.build()'
export ADAPTRA_TIMEOUT_MS=60000
timeout 600 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_stage.py -x -q > gpurun_out/r02u_pytest_stage.txt 2>&1; echo st rc=$?
tail -3 gpurun_out/r02u_pytest_stage.txt
for rep in 1 2 3; do
  for v in 1 0; do
    ADAPTRA_DB_FUSED=$v OPB_WN=4 REPS=10 timeout 300 python scripts/op_bench.py > gpurun_out/r02u_opb_db${v}_$rep.json 2>&1; echo opb$v $rep rc=$?
  done
done
for rep in 1 2 3; do
  for v in 1 0; do
    ADAPTRA_DB_FUSED=$v timeout 600 python bench.py --arms adaptive --no-e2e --no-cpu --steps 8 --warmup 3 > gpurun_out/r02u_bench_db${v}_$rep.json 2>/dev/null; echo bench$v $rep rc=$?
  done
done
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02u_pytest_gpu.txt 2>&1; echo all rc=$?
tail -3 gpurun_out/r02u_pytest_gpu.txt
