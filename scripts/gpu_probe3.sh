mkdir -p gpurun_out
./scripts/probes/launch_probe > gpurun_out/launch_probe.log 2>&1
timeout 900 python -m pytest tests/test_gpu_sweep.py -x -q -m gpu > gpurun_out/pytest_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sweep.log
timeout 600 python bench.py --workload cfg5 --steps 10 --warmup 3 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
TP_PROFILE_HOST=1 timeout 300 python scripts/e2e_probe.py > gpurun_out/e2e.log 2>&1
echo done
