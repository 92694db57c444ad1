set -x
python -c 'import __graft_entry__ as g; g.build()'
(cd _base && git checkout -q --detach 2>/dev/null; true)
export ADAPTRA_TIMEOUT_MS=60000
timeout 900 python -m pytest tests/test_gpu_stage.py tests/test_gpu_fullsize.py -x -q > gpurun_out/r02gg_pytest.txt 2>&1; echo st rc=$?
tail -2 gpurun_out/r02gg_pytest.txt
ADAPTRA_ATTN_FWD_WARPS=16 timeout 900 python -m pytest tests/test_gpu_stage.py -x -q > gpurun_out/r02gg_pytest_w16.txt 2>&1; echo w16 rc=$?
tail -2 gpurun_out/r02gg_pytest_w16.txt
for rep in 1 2 3; do
  for v in 8 16; do
    ADAPTRA_ATTN_FWD_WARPS=$v REPS=10 timeout 300 python scripts/op_bench.py > gpurun_out/r02gg_opb_w${v}_$rep.json 2>&1; echo opb $v $rep rc=$?
  done
done
