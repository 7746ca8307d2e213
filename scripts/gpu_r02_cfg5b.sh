# cfg5 batch modes: parity tests, bench per mode, launch list, --set full of the mode-5 kernels.
mkdir -p gpurun_out
TAG=${TAG:-r02e}
timeout 1200 python -m pytest tests/test_gpu_sweep.py -x -q > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}.log
for M in 5 4 0; do
TP_BATCH_MODE=$M timeout 600 python bench.py --workload cfg5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cfg5_m${M}_${TAG}.json 2> gpurun_out/cfg5_m${M}_${TAG}.err
done
CMD5="python bench.py --workload cfg5 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 3"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv \
  --log-file gpurun_out/launches_cfg5_${TAG}.csv $CMD5 > gpurun_out/ncu_launches5_${TAG}.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fused_batch --launch-skip 6 --launch-count 2 \
  -o gpurun_out/batch_${TAG} -f $CMD5 > gpurun_out/ncu_batch_${TAG}.log 2>&1
echo done
