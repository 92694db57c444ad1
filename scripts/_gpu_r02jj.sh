set -x
python -c 'import __graft_entry__ as g; g.build()'
export ADAPTRA_TIMEOUT_MS=60000
timeout 900 python -m pytest tests/test_gpu_stage.py tests/test_gpu_fullsize.py tests/test_gpu_pipeline.py -x -q > gpurun_out/r02jj_pytest.txt 2>&1; echo st rc=$?
tail -1 gpurun_out/r02jj_pytest.txt
for rep in 1 2 3; do
  for v in 0 1; do
    ADAPTRA_ATTN_POLY=$v REPS=10 timeout 300 python scripts/op_bench.py > gpurun_out/r02jj_opb_p${v}_$rep.json 2>&1; echo opb $v $rep rc=$?
  done
done
ADAPTRA_ATTN_DIAG=512 REPS=1 timeout 300 python scripts/op_bench.py > /dev/null 2> gpurun_out/r02jj_trace.txt; grep "fwd g" gpurun_out/r02jj_trace.txt | head -12
for rep in 1 2; do timeout 600 python bench.py --arms adaptive --no-e2e --no-cpu --steps 8 --warmup 3 > gpurun_out/r02jj_bench_$rep.json 2>/dev/null; echo bench rc=$?; done
