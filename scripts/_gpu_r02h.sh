set -x
python -c 'import __graft_entry__ as g; g.build()'
export ADAPTRA_TIMEOUT_MS=60000
timeout 300 python -m pytest tests/test_gpu_stage.py -x -q -k "BF16 or 1-" > gpurun_out/r02_pytest_pp_stage.txt 2>&1; echo stage rc=$?
tail -3 gpurun_out/r02_pytest_pp_stage.txt
timeout 300 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/r02_pytest_pp_full.txt 2>&1; echo full rc=$?
tail -3 gpurun_out/r02_pytest_pp_full.txt
for v in "" "ADAPTRA_ATTN_FWD=single" "ADAPTRA_COLSUM_GROUPED=0"; do
  env $v REPS=8 timeout 300 python scripts/op_bench.py >> gpurun_out/r02_op_bench_pp.jsonl 2>&1
  env $v REPS=8 timeout 300 python scripts/op_bench.py >> gpurun_out/r02_op_bench_pp.jsonl 2>&1
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02_pytest_gpu_6.txt 2>&1; echo pytest rc=$?
tail -3 gpurun_out/r02_pytest_gpu_6.txt
timeout 1200 python bench.py --arms adaptive,zb --no-cpu > gpurun_out/r02_bench_6.json 2> gpurun_out/r02_bench_6.err; echo bench rc=$?
