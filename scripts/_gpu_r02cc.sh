set -x
python -c 'import __graft_entry__ as g; g.build()'
export ADAPTRA_TIMEOUT_MS=60000
ADAPTRA_ATTN_FWD=ptmem timeout 900 python -m pytest tests/test_gpu_stage.py tests/test_gpu_fullsize.py tests/test_gpu_gemm.py -x -q > gpurun_out/r02cc_pytest_ptmem.txt 2>&1; echo pt rc=$?
tail -2 gpurun_out/r02cc_pytest_ptmem.txt
for rep in 1 2 3; do
  for v in default ptmem; do
    ADAPTRA_ATTN_FWD=$v REPS=10 timeout 300 python scripts/op_bench.py > gpurun_out/r02cc_opb_${v}_$rep.json 2>&1; echo opb $v $rep rc=$?
  done
done
for rep in 1 2; do
  for v in default ptmem; do
    ADAPTRA_ATTN_FWD=$v timeout 600 python bench.py --arms adaptive --no-e2e --no-cpu --steps 8 --warmup 3 > gpurun_out/r02cc_bench_${v}_$rep.json 2>/dev/null; echo bench $v $rep rc=$?
  done
done
