set -x
python -c 'import __graft_entry__ as g; g.build()'
for v in "" "ADAPTRA_ATTN_FWD_WARPS=16" "OPB_W2=1" "ADAPTRA_COLSUM_GROUPED=1"; do
  env $v REPS=8 timeout 300 python scripts/op_bench.py >> gpurun_out/r02_op_bench_ab.jsonl 2>&1
  env $v REPS=8 timeout 300 python scripts/op_bench.py >> gpurun_out/r02_op_bench_ab.jsonl 2>&1
done
timeout 600 python bench.py --S 8 --N 8 --steps 1 --warmup 1 --arms adaptive --no-e2e --no-cpu > gpurun_out/r02_ll_plain.json 2>&1 && \
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/r02_launches_s8n8.csv python bench.py --S 8 --N 8 --steps 1 --warmup 1 --arms adaptive --no-e2e --no-cpu > gpurun_out/r02_ll_ncu.log 2>&1; echo ncu rc=$?
