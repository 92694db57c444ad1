set -x
python -c 'import __graft_entry__ as g; g.build()'
timeout 900 python -m pytest tests/test_gpu_stage.py tests/test_gpu_pipeline.py -x -q > gpurun_out/r02_pytest_gpu_9a.txt 2>&1; echo pa rc=$?
tail -3 gpurun_out/r02_pytest_gpu_9a.txt
for rep in 1 2; do
  for v in "ADAPTRA_W_GROUP=4" "ADAPTRA_W_GROUP=2"; do
    env $v timeout 600 python bench.py --arms adaptive --no-e2e --no-cpu --steps 8 --warmup 3 > gpurun_out/r02o_${v}_$rep.json 2>/dev/null; echo $v $rep rc=$?
  done
done
for v in "ADAPTRA_X=0" "OPB_W2=1"; do env $v REPS=8 timeout 300 python scripts/op_bench.py >> gpurun_out/r02o_op.jsonl 2>&1; done
