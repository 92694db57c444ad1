set -x
python -c 'import __graft_entry__ as g; g.build()'
export ADAPTRA_TIMEOUT_MS=60000
ADAPTRA_ATTN_FWD=sep timeout 600 python -m pytest tests/test_gpu_stage.py -x -q > gpurun_out/r02nn_pytest_sep.txt 2>&1; echo sep rc=$?
tail -3 gpurun_out/r02nn_pytest_sep.txt
ADAPTRA_ATTN_FWD=sep timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/r02nn_pytest_sep_fs.txt 2>&1; echo sepfs rc=$?
tail -1 gpurun_out/r02nn_pytest_sep_fs.txt
for rep in 1 2 3; do
  for v in default sep; do
    ADAPTRA_ATTN_FWD=$v REPS=10 timeout 200 python scripts/op_bench.py > gpurun_out/r02nn_opb_${v}_$rep.json 2>&1; echo opb $v $rep rc=$?
  done
done
ADAPTRA_ATTN_FWD=sep ADAPTRA_ATTN_DIAG=512 REPS=1 timeout 200 python scripts/op_bench.py > /dev/null 2> gpurun_out/r02nn_trace_sep.txt; grep "fwd g" gpurun_out/r02nn_trace_sep.txt | head -12
