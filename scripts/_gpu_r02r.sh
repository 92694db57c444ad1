set -x
python -c 'import __graft_entry__ as g; g.build()'
export ADAPTRA_TIMEOUT_MS=60000
timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q > gpurun_out/r02r_pytest_multiproc.txt 2>&1; echo mp rc=$?
tail -3 gpurun_out/r02r_pytest_multiproc.txt
timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29631 scripts/trace_replay.py --S 4 --N 16 --compress 1 --arms adaptive,adaptive-nccl,zb-nccl --replan-log gpurun_out/r02r_replan_log.jsonl > gpurun_out/r02r_trace_full_s4_nccl.jsonl 2> gpurun_out/r02r_trace_full_s4_nccl.err; echo t4 rc=$?
tail -5 gpurun_out/r02r_trace_full_s4_nccl.err
