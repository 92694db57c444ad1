set -x
python -c 'import __graft_entry__ as g; g.build()'
export ADAPTRA_TIMEOUT_MS=60000
ADAPTRA_GEMM_MC=1 timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/r02q_pytest_gemm_mc.txt 2>&1; echo gemm_mc rc=$?
tail -3 gpurun_out/r02q_pytest_gemm_mc.txt
ADAPTRA_GEMM_MC=1 timeout 300 python -m pytest tests/test_gpu_stage.py tests/test_gpu_fullsize.py -x -q > gpurun_out/r02q_pytest_stage_mc.txt 2>&1; echo stage_mc rc=$?
tail -3 gpurun_out/r02q_pytest_stage_mc.txt
ADAPTRA_GEMM_MC=1 REPS=20 timeout 300 python scripts/gemm_bench.py > gpurun_out/r02q_gemm_mc.jsonl 2>&1; echo b1 rc=$?
REPS=20 timeout 300 python scripts/gemm_bench.py > gpurun_out/r02q_gemm_base.jsonl 2>&1; echo b2 rc=$?
for rep in 1 2; do
  for v in "ADAPTRA_X=0" "ADAPTRA_LOOKAHEAD=2" "ADAPTRA_LOOKAHEAD=5" "CUDA_DEVICE_MAX_CONNECTIONS=16" "ADAPTRA_INORDER_QUEUE=2"; do
    env $v timeout 600 python bench.py --arms adaptive --no-e2e --no-cpu --steps 8 --warmup 3 > gpurun_out/r02p_${v}_$rep.json 2>/dev/null; echo $v $rep rc=$?
  done
done
