mkdir -p gpurun_out
MODE=full python scripts/ncu_probe.py > gpurun_out/ncu_probe_plain.log 2>&1 && \
MODE=full ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --csv \
  --log-file gpurun_out/launches_probe.csv python scripts/ncu_probe.py > gpurun_out/ncu_l.log 2>&1
echo done
