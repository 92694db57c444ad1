set -x
python -c 'import __graft_entry__ as g; g.build()'
export ADAPTRA_TIMEOUT_MS=60000
T='tests/test_gpu_fullsize.py::test_full_size_block_fbw[2048-8192-16-1-False-2]'
timeout 300 python -m pytest "$T" -x -q > gpurun_out/r02v_default.txt 2>&1; echo a rc=$?
ADAPTRA_DB_FUSED=0 timeout 300 python -m pytest "$T" -x -q > gpurun_out/r02v_dbfused0.txt 2>&1; echo b rc=$?
ADAPTRA_GEMM_GROUPED=0 timeout 300 python -m pytest "$T" -x -q > gpurun_out/r02v_grouped0.txt 2>&1; echo c rc=$?
grep -h "AssertionError" gpurun_out/r02v_*.txt | cut -c1-600
