set -x
python -c 'import __graft_entry__ as g; g.build()'
export ADAPTRA_TIMEOUT_MS=60000
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29651 scripts/mp_check.py > gpurun_out/r02x_mp_check.txt 2>&1; echo mp rc=$?
grep -E "probe|FAIL" gpurun_out/r02x_mp_check.txt | head
grep -c " OK" gpurun_out/r02x_mp_check.txt
timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29652 scripts/trace_replay.py --S 4 --N 16 --compress 1 --arms adaptive,zb-nccl,adaptive-nccl,1f1b-nccl,zb > gpurun_out/r02x_trace_full_s4_nccl.jsonl 2> gpurun_out/r02x_trace_full_s4_nccl.err; echo t4 rc=$?
tail -3 gpurun_out/r02x_trace_full_s4_nccl.err
