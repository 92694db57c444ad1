set -x
python -c 'import __graft_entry__ as g; g.build()'
ONLY=F_o REPS=2 timeout 300 python scripts/gemm_bench.py > gpurun_out/r02j_gemm_F_o.plain.log 2>&1 && \
ONLY=F_o REPS=2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 3 -c 1 -o gpurun_out/r02j_ncu_gemm_F_o_src python scripts/gemm_bench.py > gpurun_out/r02j_ncu_gemm.log 2>&1; echo ncu1 rc=$?
LAYERS=1 NMB=2 REPS=1 timeout 300 python scripts/op_bench.py > gpurun_out/r02j_op.plain.log 2>&1 && \
LAYERS=1 NMB=2 REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd -s 2 -c 1 -o gpurun_out/r02j_ncu_attn_fwd_src python scripts/op_bench.py > gpurun_out/r02j_ncu_attn.log 2>&1; echo ncu2 rc=$?
for rep in 1 2 3; do
  for v in "ADAPTRA_X=0" "ADAPTRA_COLSUM_GROUPED=0" "ADAPTRA_W_PAIRS=0"; do
    env $v timeout 600 python bench.py --arms adaptive --no-e2e --no-cpu --steps 8 --warmup 3 > gpurun_out/r02k_${v}_$rep.json 2>/dev/null; echo $v $rep rc=$?
  done
done
