set -x
python -c 'import __graft_entry__ as g; g.build()'
for rep in 1 2; do
  for v in "ADAPTRA_X=0" "ADAPTRA_LOOKAHEAD=2" "ADAPTRA_LOOKAHEAD=5" "CUDA_DEVICE_MAX_CONNECTIONS=16" "ADAPTRA_INORDER_QUEUE=2"; do
    env $v timeout 600 python bench.py --arms adaptive --no-e2e --no-cpu --steps 8 --warmup 3 > gpurun_out/r02p_${v}_$rep.json 2>/dev/null; echo $v $rep rc=$?
  done
done
