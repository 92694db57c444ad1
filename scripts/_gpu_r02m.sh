set -x
python -c 'import __graft_entry__ as g; g.build()'
for rep in 1 2; do
  for v in 0 74 100 120; do
    ADAPTRA_GEMM_SMS=$v timeout 600 python bench.py --arms adaptive --no-e2e --no-cpu --steps 8 --warmup 3 > gpurun_out/r02m_sms${v}_$rep.json 2>/dev/null; echo $v $rep rc=$?
  done
done
