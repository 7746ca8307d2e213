mkdir -p gpurun_out
MODE=pairs python scripts/ncu_probe.py > gpurun_out/ncu_probe_plain.log 2>&1 && \
MODE=pairs ncu --set full --import-source on --clock-control none -k regex:fused_kernel --launch-skip 4 --launch-count 1 \
  -o gpurun_out/fused_pairs -f python scripts/ncu_probe.py > gpurun_out/ncu_pairs.log 2>&1
MODE=full ncu --set full --import-source on --clock-control none -k regex:fused_kernel --launch-skip 4 --launch-count 1 \
  -o gpurun_out/fused_full -f python scripts/ncu_probe.py > gpurun_out/ncu_full.log 2>&1
echo done
