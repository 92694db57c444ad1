set -x
python -c 'import __graft_entry__ as g; g.build()'
export ADAPTRA_TIMEOUT_MS=60000
for rep in 1 2 3; do
  for v in default smem; do
    ADAPTRA_ATTN_FWD=$v timeout 200 python bench.py --no-e2e --no-cpu --steps 8 --warmup 3 > gpurun_out/r02ss_bench_${v}_$rep.json 2> gpurun_out/r02ss_bench_${v}_$rep.err; echo bench $v $rep rc=$?
  done
done
