set -x
python -c 'import __graft_entry__ as g; g.build()'
timeout 1200 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_transfer.py -x -q > gpurun_out/r02_pytest_multigpu_final.txt 2>&1; echo pytest rc=$?
tail -3 gpurun_out/r02_pytest_multigpu_final.txt
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29631 bench.py --gpus 4 > gpurun_out/r02_bench_4gpu_final.json 2> gpurun_out/r02_bench_4gpu_final.err; echo b4 rc=$?
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29632 bench.py --gpus 2 > gpurun_out/r02_bench_2gpu_final.json 2> gpurun_out/r02_bench_2gpu_final.err; echo b2 rc=$?
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29633 bench.py --gpus 4 --model 7b --no-cpu --arms adaptive,zb,1f1b,zb-inorder > gpurun_out/r02_bench_4gpu_7b.json 2> gpurun_out/r02_bench_4gpu_7b.err; echo b7 rc=$?
tail -2 gpurun_out/r02_bench_4gpu_7b.err
