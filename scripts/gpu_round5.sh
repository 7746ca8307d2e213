mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_price.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/pytest_gpu5.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu5.log
timeout 600 python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5_groups.json 2> gpurun_out/bench_cfg5_groups.err
TP_BATCH_NO_GROUPS=1 timeout 600 python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5_nogroups.json 2> gpurun_out/bench_cfg5_nogroups.err
TP_PROFILE_HOST=1 timeout 300 python scripts/sweep_probe.py 2>&1 | grep -v "tp host" > gpurun_out/sweep_probe.log
echo done
