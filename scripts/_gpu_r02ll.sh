set -x
python -c 'import __graft_entry__ as g; g.build()'
export ADAPTRA_TIMEOUT_MS=60000
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29681 bench.py --gpus 4 --S 4 --N 16 --steps 6 --warmup 3 > gpurun_out/r02ll_bench_4gpu_s4.json 2> gpurun_out/r02ll_bench_4gpu_s4.err; echo b rc=$?
tail -c 1500 gpurun_out/r02ll_bench_4gpu_s4.json
tail -3 gpurun_out/r02ll_bench_4gpu_s4.err
