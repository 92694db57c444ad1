set -x
python -c 'import __graft_entry__ as g; g.build()'
export ADAPTRA_TIMEOUT_MS=60000
ADAPTRA_ATTN_FWD=s2 timeout 600 python -m pytest tests/test_gpu_stage.py -x -q > gpurun_out/r02pp_pytest_s2.txt 2>&1; echo s2 rc=$?
tail -3 gpurun_out/r02pp_pytest_s2.txt
ADAPTRA_ATTN_FWD=s2 timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/r02pp_pytest_s2_fs.txt 2>&1; echo s2fs rc=$?
tail -1 gpurun_out/r02pp_pytest_s2_fs.txt
for rep in 1 2 3; do
  for v in default s2; do
    ADAPTRA_ATTN_FWD=$v REPS=10 timeout 200 python scripts/op_bench.py > gpurun_out/r02pp_opb_${v}_$rep.json 2>&1; echo opb $v $rep rc=$?
  done
done
ADAPTRA_ATTN_FWD=s2 ADAPTRA_ATTN_DIAG=512 REPS=1 timeout 200 python scripts/op_bench.py > /dev/null 2> gpurun_out/r02pp_trace_s2.txt; grep "fwd g" gpurun_out/r02pp_trace_s2.txt | head -12
