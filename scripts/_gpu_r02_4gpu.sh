set -x
nvidia-smi --query-gpu=index,name,memory.total --format=csv
python -c 'import __graft_entry__ as g; g.build()'
timeout 1200 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_transfer.py -x -q > gpurun_out/r02_pytest_multigpu.txt 2>&1; echo pytest rc=$?
tail -4 gpurun_out/r02_pytest_multigpu.txt
REPS=20 timeout 300 python scripts/direct_nvlink.py > gpurun_out/r02_direct_nvlink.json 2>&1 && \
REPS=1 timeout 600 ncu --metrics nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemm_tc --csv --log-file gpurun_out/r02_ncu_direct_nvlink.csv python scripts/direct_nvlink.py > gpurun_out/r02_ncu_direct_nvlink.log 2>&1; echo ncu rc=$?
timeout 300 python scripts/nvlink_bench.py > gpurun_out/r02_nvlink_bench.jsonl 2>&1; echo nvl rc=$?
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 4 --steps 10 --warmup 3 --replan-log gpurun_out/r02_replan_log_c3_s8_4gpu.jsonl > gpurun_out/r02_bench_4gpu.json 2> gpurun_out/r02_bench_4gpu.err; echo bench4 rc=$?
tail -3 gpurun_out/r02_bench_4gpu.err
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 4 --S 4 --N 16 --steps 10 --warmup 3 --no-cpu --arms adaptive,zb,1f1b,zb-inorder,zb-nccl,1f1b-nccl,adaptive-deleg > gpurun_out/r02_bench_4gpu_c1_nccl.json 2> gpurun_out/r02_bench_4gpu_c1_nccl.err; echo bench_c1 rc=$?
tail -3 gpurun_out/r02_bench_4gpu_c1_nccl.err
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu > gpurun_out/r02_bench_2gpu.json 2> gpurun_out/r02_bench_2gpu.err; echo bench2 rc=$?
