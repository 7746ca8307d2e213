# Round profile: bench (no profiler), then the ncu launch list and one
# --set full capture of the fused kernel from the same bench command.
mkdir -p gpurun_out
TAG=${TAG:-r01}
python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 3"
$CMD > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launches_${TAG}.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:fused_kernel --launch-skip 3 --launch-count 1 \
  -o gpurun_out/fused_${TAG} -f $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo done
