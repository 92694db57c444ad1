set -x
python -c 'import __graft_entry__ as g; g.build()'
export ADAPTRA_TIMEOUT_MS=60000
timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q > gpurun_out/r02ee_pytest_multiproc.txt 2>&1; echo mp rc=$?
tail -2 gpurun_out/r02ee_pytest_multiproc.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29671 scripts/mp_check.py > gpurun_out/r02ee_mp_check.txt 2>&1; echo mpc rc=$?
grep -E "nccl|probe" gpurun_out/r02ee_mp_check.txt | head -12
REPS=1 NMB=4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 3 -c 1 -o gpurun_out/r02ee_ncu_attn_fwd python scripts/op_bench.py > gpurun_out/r02ee_ncu_attn_fwd.log 2>&1; echo ncuf rc=$?
REPS=1 NMB=4 timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_bwd -s 3 -c 1 -o gpurun_out/r02ee_ncu_attn_bwd python scripts/op_bench.py > gpurun_out/r02ee_ncu_attn_bwd.log 2>&1; echo ncub rc=$?
ADAPTRA_ATTN_FWD=qtmem timeout 900 python -m pytest tests/test_gpu_stage.py tests/test_gpu_fullsize.py -x -q > gpurun_out/r02ee_pytest_qtmem.txt 2>&1; echo qt rc=$?
tail -2 gpurun_out/r02ee_pytest_qtmem.txt
for rep in 1 2 3; do
  for v in default qtmem; do
    ADAPTRA_ATTN_FWD=$v REPS=10 timeout 300 python scripts/op_bench.py > gpurun_out/r02ee_opb_${v}_$rep.json 2>&1; echo opb $v $rep rc=$?
  done
done
