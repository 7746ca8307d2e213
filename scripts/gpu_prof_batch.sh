mkdir -p gpurun_out
CMD="python bench.py --workload cfg5 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 3"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fused_batch --launch-skip 3 --launch-count 1 \
  -o gpurun_out/batch_groups -f $CMD > gpurun_out/ncu_bg.log 2>&1
TP_BATCH_NO_GROUPS=1 timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum,l1tex__t_bytes_pipe_lsu_mem_local_op_st.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:fused_batch --launch-skip 3 --launch-count 1 \
  $CMD > gpurun_out/ncu_bn.log 2>&1
echo done
