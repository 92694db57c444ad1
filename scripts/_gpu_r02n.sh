set -x
python -c 'import __graft_entry__ as g; g.build()'
for rep in 1 2; do
  for v in "ADAPTRA_X=0" "ADAPTRA_ATTN_SMS=74" "ADAPTRA_GEMM_SMS=56" "ADAPTRA_GEMM_SMS=37"; do
    env $v timeout 600 python bench.py --arms adaptive --no-e2e --no-cpu --steps 8 --warmup 3 > gpurun_out/r02n_${v}_$rep.json 2>/dev/null; echo $v $rep rc=$?
  done
done
REPS=20 timeout 300 python scripts/gemm_bench.py > gpurun_out/r02n_gemm.jsonl 2>&1
