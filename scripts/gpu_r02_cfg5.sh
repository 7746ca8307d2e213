# cfg5 iteration: sweep parity tests, bench A/B (op lists vs class tables), launch list, one --set full capture.
mkdir -p gpurun_out
TAG=${TAG:-r02d}
timeout 900 python -m pytest tests/test_gpu_sweep.py -x -q > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}.log
timeout 600 python bench.py --workload cfg5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cfg5_${TAG}.json 2> gpurun_out/cfg5_${TAG}.err
TP_BATCH_OPLISTS=0 timeout 600 python bench.py --workload cfg5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cfg5_tables_${TAG}.json 2> gpurun_out/cfg5_tables_${TAG}.err
CMD5="python bench.py --workload cfg5 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 3"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 40 --csv \
  --log-file gpurun_out/launches_cfg5_${TAG}.csv $CMD5 > gpurun_out/ncu_launches5_${TAG}.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fused_batch --launch-skip 3 --launch-count 1 \
  -o gpurun_out/batch_${TAG} -f $CMD5 > gpurun_out/ncu_batch_${TAG}.log 2>&1
echo done
