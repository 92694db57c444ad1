set -x
python -c 'import __graft_entry__ as g; g.build()'
export ADAPTRA_TIMEOUT_MS=60000
ADAPTRA_ATTN_FWD_WARPS=16 timeout 900 python -m pytest tests/test_gpu_stage.py tests/test_gpu_fullsize.py -x -q > gpurun_out/r02ff_pytest_w16.txt 2>&1; echo w16 rc=$?
tail -2 gpurun_out/r02ff_pytest_w16.txt
for rep in 1 2 3; do
  for v in 8 16; do
    ADAPTRA_ATTN_FWD_WARPS=$v REPS=10 timeout 300 python scripts/op_bench.py > gpurun_out/r02ff_opb_w${v}_$rep.json 2>&1; echo opb $v $rep rc=$?
  done
done
