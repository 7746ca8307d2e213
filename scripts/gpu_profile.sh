mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 3"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"build_kernel_warp|expand_kernel" -s 2 -c 2 -o gpurun_out/prof_v2 $CMD > gpurun_out/ncu_v2.log 2>&1
echo done
