# Round-2 full check: GPU test suite, the default bench line (all blocks), cfg5 per batch mode,
# launch list + --set full capture of the batch kernels.
mkdir -p gpurun_out
TAG=${TAG:-r02f}
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
for M in 5 4; do
TP_BATCH_MODE=$M timeout 600 python bench.py --workload cfg5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cfg5_m${M}_${TAG}.json 2> gpurun_out/cfg5_m${M}_${TAG}.err
done
CMD5="python bench.py --workload cfg5 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 3"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"batch|infer" -c 40 --csv \
  --log-file gpurun_out/launches_cfg5_${TAG}.csv $CMD5 > gpurun_out/ncu_launches5_${TAG}.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fused_batch --launch-skip 6 --launch-count 2 \
  -o gpurun_out/batch_${TAG} -f $CMD5 > gpurun_out/ncu_batch_${TAG}.log 2>&1
echo done
