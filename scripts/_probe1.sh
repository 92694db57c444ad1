nvidia-smi --query-gpu=name,memory.total,memory.used --format=csv
python -c "import torch; print(torch.cuda.mem_get_info())"
timeout 900 python bench.py --S 8 --N 32 --steps 3 --warmup 3 --arms adaptive,zb --no-cpu --no-e2e > gpurun_out/probe_s8n32.json 2> gpurun_out/probe_s8n32.err; echo rc=$?
tail -5 gpurun_out/probe_s8n32.err
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r2_start.txt 2>&1; echo rc=$?
tail -5 gpurun_out/pytest_gpu_r2_start.txt
