set -x
python -c 'import __graft_entry__ as g; g.build()'
timeout 1200 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_stage.py tests/test_gpu_pipeline.py -x -q > gpurun_out/r02_pytest_gpu_2.txt 2>&1; echo pytest rc=$?
tail -5 gpurun_out/r02_pytest_gpu_2.txt
nvidia-smi --query-gpu=memory.used,memory.total --format=csv
timeout 900 python bench.py --S 8 --N 32 --steps 4 --warmup 3 --arms adaptive,zb --no-cpu --no-e2e > gpurun_out/r02_probe_s8n32.json 2> gpurun_out/r02_probe_s8n32.err; echo bench rc=$?
tail -4 gpurun_out/r02_probe_s8n32.err
export ADAPTRA_TIMEOUT_MS=600000
timeout 1200 compute-sanitizer --tool memcheck --launch-timeout 600 python -m pytest tests/test_gpu_stage.py -x -q -k "gpt and 256 and 1024" > gpurun_out/r02_sanitizer_memcheck_stage.txt 2>&1; echo memcheck rc=$?
tail -5 gpurun_out/r02_sanitizer_memcheck_stage.txt
timeout 1500 compute-sanitizer --tool racecheck --launch-timeout 600 python -m pytest tests/test_gpu_stage.py -x -q -k "gpt and 256 and 1024 and not True" > gpurun_out/r02_sanitizer_racecheck_stage.txt 2>&1; echo racecheck rc=$?
tail -5 gpurun_out/r02_sanitizer_racecheck_stage.txt
