set -x
python -c 'import __graft_entry__ as g; g.build()'
export ADAPTRA_TIMEOUT_MS=60000
ADAPTRA_ATTN_FWD=qtmem ADAPTRA_ATTN_DIAG=512 REPS=1 timeout 300 python scripts/op_bench.py > /dev/null 2> gpurun_out/r02mm_trace_qt.txt; grep "fwd g" gpurun_out/r02mm_trace_qt.txt | head -12
ADAPTRA_ATTN_FWD=smem ADAPTRA_ATTN_DIAG=512 REPS=1 timeout 300 python scripts/op_bench.py > /dev/null 2> gpurun_out/r02mm_trace_smem.txt; grep "fwd g" gpurun_out/r02mm_trace_smem.txt | head -12
