# Round evidence on one GPU: test suite, default bench (all blocks), reference arm,
# cfg5 chunk variants, launch list + one --set full capture of fused_kernel and the batch kernels.
mkdir -p gpurun_out
TAG=${TAG:-r02}
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}.log
timeout 1200 ./oracle/_ref/adapter_parity > gpurun_out/adapter_parity_${TAG}.log 2>&1; echo "rc=$?" >> gpurun_out/adapter_parity_${TAG}.log
./oracle/_ref/export_parity --big > gpurun_out/export_parity_${TAG}.log 2>&1; echo "rc=$?" >> gpurun_out/export_parity_${TAG}.log
python scripts/fan_probe.py > gpurun_out/fan_${TAG}.log 2>&1
python scripts/class_probe.py > gpurun_out/class_${TAG}.log 2>&1
TP_PROFILE_HOST=1 timeout 300 python scripts/e2e_probe.py > gpurun_out/e2e_probe_${TAG}.log 2>&1
TP_PROFILE_HOST=1 timeout 300 python scripts/sweep_probe.py > gpurun_out/sweep_probe_${TAG}.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err
timeout 900 python bench.py --impl reference --workload cfg5 --steps 3 > gpurun_out/bench_ref_cfg5_${TAG}.json 2> gpurun_out/bench_ref_cfg5_${TAG}.err
for C in 12 24; do TP_SWEEP_CHUNKS=$C timeout 600 python bench.py --workload cfg5 --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 6 > gpurun_out/cfg5_c${C}_${TAG}.json 2>/dev/null; done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 3 --no-sweep --no-configs"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launches_${TAG}.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fused_kernel --launch-skip 3 --launch-count 1 \
  -o gpurun_out/fused_${TAG} -f $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
CMD5="python bench.py --workload cfg5 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 3"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"batch|infer" -c 60 --csv \
  --log-file gpurun_out/launches_cfg5_${TAG}.csv $CMD5 > gpurun_out/ncu_launches5_${TAG}.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"fused_batch|infer" --launch-skip 9 --launch-count 3 \
  -o gpurun_out/batch_${TAG} -f $CMD5 > gpurun_out/ncu_batch_${TAG}.log 2>&1
echo done
