set -x
python -c 'import __graft_entry__ as g; g.build()'
export ADAPTRA_TIMEOUT_MS=60000
ADAPTRA_ATTN_DIAG=512 REPS=1 timeout 300 python scripts/op_bench.py > gpurun_out/r02hh_trace.json 2> gpurun_out/r02hh_trace.txt; echo tr rc=$?
grep "fwd g" gpurun_out/r02hh_trace.txt | head -40
for rep in 1 2; do REPS=10 timeout 300 python scripts/op_bench.py > gpurun_out/r02hh_opb_$rep.json 2>&1; echo opb rc=$?; done
timeout 600 python -m pytest tests/test_gpu_stage.py -x -q > gpurun_out/r02hh_pytest.txt 2>&1; echo st rc=$?
tail -1 gpurun_out/r02hh_pytest.txt
