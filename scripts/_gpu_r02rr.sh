set -x
python -c 'import __graft_entry__ as g; g.build()'
export ADAPTRA_TIMEOUT_MS=60000
for rep in 1 2; do
  timeout 300 python bench.py > gpurun_out/r02rr_bench_default_$rep.json 2> gpurun_out/r02rr_bench_default_$rep.err; echo bench $rep rc=$?
done
ADAPTRA_ATTN_FWD=smem timeout 300 python bench.py --no-cpu > gpurun_out/r02rr_bench_smem.json 2> gpurun_out/r02rr_bench_smem.err; echo bench smem rc=$?
nvidia-smi --query-gpu=clocks.sm,clocks_throttle_reasons.active --format=csv
