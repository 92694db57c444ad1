set -x
python -c 'import __graft_entry__ as g; g.build()'
export ADAPTRA_TIMEOUT_MS=60000
timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q > gpurun_out/r02bb_pytest_multiproc.txt 2>&1; echo mp rc=$?
tail -2 gpurun_out/r02bb_pytest_multiproc.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29661 bench.py --gpus 4 --steps 8 --warmup 3 > gpurun_out/r02bb_bench_4gpu.json 2> gpurun_out/r02bb_bench_4gpu.err; echo b4 rc=$?
CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29662 bench.py --gpus 2 --steps 8 --warmup 3 > gpurun_out/r02bb_bench_2gpu.json 2> gpurun_out/r02bb_bench_2gpu.err; echo b2 rc=$?
timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29663 scripts/trace_replay.py --S 4 --N 16 --compress 1 --arms adaptive,zb,zb-nccl,adaptive-nccl,1f1b-nccl --replan-log gpurun_out/r02bb_replan_log_c3_full_s4.jsonl > gpurun_out/r02bb_trace_full_s4_nccl.jsonl 2> gpurun_out/r02bb_trace_full_s4_nccl.err; echo t4 rc=$?
timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29664 scripts/stage_sweep.py > gpurun_out/r02bb_stage_sweep_c4_4gpu.jsonl 2> gpurun_out/r02bb_stage_sweep.err; echo sw rc=$?
tail -2 gpurun_out/r02bb_stage_sweep.err
