set -x
python -c 'import __graft_entry__ as g; g.build()'
export ADAPTRA_TIMEOUT_MS=60000
ADAPTRA_ATTN_POLY=2 timeout 600 python -m pytest tests/test_gpu_stage.py tests/test_gpu_fullsize.py -x -q > gpurun_out/r02s_pytest_poly2.txt 2>&1; echo poly2 rc=$?
tail -3 gpurun_out/r02s_pytest_poly2.txt
for rep in 1 2 3; do
  for v in 0 1 2; do
    ADAPTRA_ATTN_POLY=$v REPS=10 timeout 300 python scripts/op_bench.py > gpurun_out/r02s_opb_poly${v}_$rep.json 2>&1; echo poly$v $rep rc=$?
  done
done
for rep in 1 2; do
  for v in 0 2; do
    ADAPTRA_ATTN_POLY=$v timeout 600 python bench.py --arms adaptive --no-e2e --no-cpu --steps 8 --warmup 3 > gpurun_out/r02s_bench_poly${v}_$rep.json 2>/dev/null; echo bench$v $rep rc=$?
  done
done
