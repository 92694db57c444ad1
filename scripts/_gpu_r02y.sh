set -x
python -c 'import __graft_entry__ as g; g.build()'
(cd _base && python -c 'import __graft_entry__ as g; g.build()')
export ADAPTRA_TIMEOUT_MS=60000
for rep in 1 2; do
  for wn in 0 4; do
    (cd _base && OPB_WN=$wn REPS=10 timeout 300 python scripts/op_bench.py) > gpurun_out/r02y_opb_base_wn${wn}_$rep.json 2>&1
    ADAPTRA_DB_FUSED=0 OPB_WN=$wn REPS=10 timeout 300 python scripts/op_bench.py > gpurun_out/r02y_opb_off_wn${wn}_$rep.json 2>&1
    for m in 1 2 3; do
      ADAPTRA_DB_MODE=$m OPB_WN=$wn REPS=10 timeout 300 python scripts/op_bench.py > gpurun_out/r02y_opb_m${m}_wn${wn}_$rep.json 2>&1; echo m$m wn$wn rc=$?
    done
  done
done
