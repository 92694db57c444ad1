set -x
python -c 'import __graft_entry__ as g; g.build()'
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02_pytest_gpu_7.txt 2>&1; echo pytest rc=$?
tail -3 gpurun_out/r02_pytest_gpu_7.txt
timeout 600 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/r02_smoke.txt 2>&1; echo smoke rc=$?
tail -2 gpurun_out/r02_smoke.txt
timeout 1200 python bench.py --replan-log gpurun_out/r02_replan_log_c3_s8_1gpu_b7.jsonl > gpurun_out/r02_bench_7.json 2> gpurun_out/r02_bench_7.err; echo bench rc=$?
for v in "ADAPTRA_W_PAIRS=0" "ADAPTRA_LOOKAHEAD=6" "ADAPTRA_COLSUM_GROUPED=0"; do
  env $v timeout 900 python bench.py --arms adaptive --no-e2e --no-cpu > gpurun_out/r02_bench_7_$v.json 2>/dev/null; echo $v rc=$?
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02_bench_ref.json 2>&1; echo ref rc=$?
