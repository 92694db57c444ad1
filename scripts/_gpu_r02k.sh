set -x
python -c 'import __graft_entry__ as g; g.build()'
for rep in 1 2 3; do
  for v in "ADAPTRA_X=0" "ADAPTRA_COLSUM_GROUPED=0" "ADAPTRA_W_PAIRS=0"; do
    env $v timeout 600 python bench.py --arms adaptive --no-e2e --no-cpu --steps 8 --warmup 3 > gpurun_out/r02k_${v}_$rep.json 2>/dev/null; echo $v $rep rc=$?
  done
done
