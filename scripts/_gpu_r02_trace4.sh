set -x
python -c 'import __graft_entry__ as g; g.build()'
timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29621 scripts/trace_replay.py --S 4 --N 16 --compress 1 --arms adaptive,zb,zb-nccl,1f1b-nccl,zb-inorder --replan-log gpurun_out/r02_replan_log_c3_full_s4_4gpu.jsonl > gpurun_out/r02_trace_full_s4_4gpu_nccl.jsonl 2> gpurun_out/r02_trace_full_s4_4gpu_nccl.err; echo t4 rc=$?
tail -3 gpurun_out/r02_trace_full_s4_4gpu_nccl.err
timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29622 scripts/trace_replay.py --S 8 --N 32 --compress 2 --arms adaptive,zb,zb-inorder,1f1b > gpurun_out/r02_trace_c3_s8_4gpu.jsonl 2> gpurun_out/r02_trace_c3_s8_4gpu.err; echo t8 rc=$?
tail -3 gpurun_out/r02_trace_c3_s8_4gpu.err
