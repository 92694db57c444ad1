set -x
python -c 'import __graft_entry__ as g; g.build()'
(cd _base && python -c 'import __graft_entry__ as g; g.build()')
export ADAPTRA_TIMEOUT_MS=60000
timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q > gpurun_out/r02w_pytest_fullsize.txt 2>&1; echo fs rc=$?
tail -2 gpurun_out/r02w_pytest_fullsize.txt
for rep in 1 2; do
  for wn in 0 4; do
    (cd _base && OPB_WN=$wn REPS=10 timeout 300 python scripts/op_bench.py) > gpurun_out/r02w_opb_base_wn${wn}_$rep.json 2>&1; echo base$wn rc=$?
    OPB_WN=$wn REPS=10 timeout 300 python scripts/op_bench.py > gpurun_out/r02w_opb_new_wn${wn}_$rep.json 2>&1; echo new$wn rc=$?
    ADAPTRA_DB_FUSED=0 OPB_WN=$wn REPS=10 timeout 300 python scripts/op_bench.py > gpurun_out/r02w_opb_new0_wn${wn}_$rep.json 2>&1; echo new0$wn rc=$?
  done
done
for rep in 1 2; do
  (cd _base && timeout 600 python bench.py --arms adaptive --no-e2e --no-cpu --steps 8 --warmup 3) > gpurun_out/r02w_bench_base_$rep.json 2>/dev/null; echo bb rc=$?
  timeout 600 python bench.py --arms adaptive --no-e2e --no-cpu --steps 8 --warmup 3 > gpurun_out/r02w_bench_new_$rep.json 2>/dev/null; echo bn rc=$?
done
