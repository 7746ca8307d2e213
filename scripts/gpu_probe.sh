mkdir -p gpurun_out
python scripts/phase_probe.py > gpurun_out/phase_probe.log 2>&1
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 3"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"fused_kernel" -s 1 -c 1 -o gpurun_out/prof_fused $CMD > gpurun_out/ncu_f.log 2>&1
echo done
