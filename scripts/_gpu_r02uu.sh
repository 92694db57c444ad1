set -x
python -c 'import __graft_entry__ as g; g.build()'
export ADAPTRA_TIMEOUT_MS=60000
ADAPTRA_ATTN_FWD=ptmem timeout 600 python -m pytest tests/test_gpu_stage.py -x -q > gpurun_out/r02uu_pytest_pt.txt 2>&1; echo pt rc=$?
tail -1 gpurun_out/r02uu_pytest_pt.txt
for rep in 1 2 3 4 5; do
  ADAPTRA_ATTN_FWD=ptmem timeout 200 python bench.py --no-e2e --no-cpu --steps 8 --warmup 3 > gpurun_out/r02uu_bench_pt_$rep.json 2> gpurun_out/r02uu_bench_pt_$rep.err; echo bench pt $rep rc=$?
done
