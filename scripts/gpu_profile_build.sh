mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 3"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"build_kernel" -s 1 -c 1 -o gpurun_out/prof_build $CMD > gpurun_out/ncu_b.log 2>&1
echo done
