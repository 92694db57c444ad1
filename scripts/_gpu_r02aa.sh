set -x
python -c 'import __graft_entry__ as g; g.build()'
export ADAPTRA_TIMEOUT_MS=60000
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02aa_pytest_gpu.txt 2>&1; echo all rc=$?
tail -3 gpurun_out/r02aa_pytest_gpu.txt
REPS=1 NMB=4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_grouped -s 2 -c 1 -o gpurun_out/r02aa_ncu_grouped python scripts/op_bench.py > gpurun_out/r02aa_ncu_grouped.log 2>&1; echo ncu rc=$?
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/r02aa_launches_s8n8.csv python bench.py --S 8 --N 8 --steps 1 --warmup 1 --arms adaptive --no-e2e --no-cpu > gpurun_out/r02aa_ll_ncu.log 2>&1; echo ll rc=$?
