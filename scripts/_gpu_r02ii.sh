set -x
python -c 'import __graft_entry__ as g; g.build()'
export ADAPTRA_TIMEOUT_MS=60000
ADAPTRA_ATTN_POLY=1 timeout 600 python -m pytest tests/test_gpu_stage.py tests/test_gpu_fullsize.py -x -q > gpurun_out/r02ii_pytest_p1.txt 2>&1; echo p1 rc=$?
tail -1 gpurun_out/r02ii_pytest_p1.txt
ADAPTRA_ATTN_POLY=2 timeout 600 python -m pytest tests/test_gpu_stage.py -x -q > gpurun_out/r02ii_pytest_p2.txt 2>&1; echo p2 rc=$?
tail -1 gpurun_out/r02ii_pytest_p2.txt
for rep in 1 2 3; do
  for v in 0 1 2; do
    ADAPTRA_ATTN_POLY=$v REPS=10 timeout 300 python scripts/op_bench.py > gpurun_out/r02ii_opb_p${v}_$rep.json 2>&1; echo opb $v $rep rc=$?
  done
done
ADAPTRA_ATTN_POLY=1 ADAPTRA_ATTN_DIAG=512 REPS=1 timeout 300 python scripts/op_bench.py > /dev/null 2> gpurun_out/r02ii_trace_p1.txt; grep "fwd g" gpurun_out/r02ii_trace_p1.txt | head -12
