# Round-2 iteration: GPU tests of the touched paths, the bench (all blocks), cfg5 A/B, ncu of the batch kernel.
mkdir -p gpurun_out
TAG=${TAG:-r02b}
timeout 900 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_price.py -x -q > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}.log
timeout 600 python bench.py --workload cfg5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cfg5_${TAG}.json 2> gpurun_out/cfg5_${TAG}.err
TP_BATCH_OPLISTS=0 timeout 600 python bench.py --workload cfg5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cfg5_groups_${TAG}.json 2> gpurun_out/cfg5_groups_${TAG}.err
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
CMD5="python bench.py --workload cfg5 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 3"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"batch|infer" -c 60 --csv \
  --log-file gpurun_out/launches_cfg5_${TAG}.csv $CMD5 > gpurun_out/ncu_launches5_${TAG}.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fused_batch --launch-skip 3 --launch-count 1 \
  -o gpurun_out/batch_${TAG} -f $CMD5 > gpurun_out/ncu_batch_${TAG}.log 2>&1
echo done
