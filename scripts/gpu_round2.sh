mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/pytest_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sweep.log

timeout 600 python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5_narrow.json 2> gpurun_out/bench_cfg5_narrow.err
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
TP_PROFILE_HOST=1 timeout 300 python scripts/e2e_probe.py > gpurun_out/e2e.log 2>&1
echo done
