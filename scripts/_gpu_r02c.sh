set -x
python -c 'import __graft_entry__ as g; g.build()'
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02_pytest_gpu_3.txt 2>&1; echo pytest rc=$?
tail -5 gpurun_out/r02_pytest_gpu_3.txt
timeout 1200 python bench.py --replan-log gpurun_out/r02_replan_log_c3_s8_1gpu.jsonl > gpurun_out/r02_bench_3.json 2> gpurun_out/r02_bench_3.err; echo bench rc=$?
tail -3 gpurun_out/r02_bench_3.err
for sh in F_o F_fc1 B_qkv; do
  ONLY=$sh REPS=2 timeout 300 python scripts/gemm_bench.py > gpurun_out/r02_gemm_$sh.plain.log 2>&1 && \
  ONLY=$sh REPS=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 3 -c 1 -o gpurun_out/r02_ncu_gemm_$sh python scripts/gemm_bench.py > gpurun_out/r02_ncu_gemm_$sh.log 2>&1; echo ncu $sh rc=$?
done
