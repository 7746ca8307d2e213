mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_sweep.py -x -q -m gpu > gpurun_out/pytest_gpu10.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu10.log
for i in 1 2; do timeout 600 python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/bench_cfg5_ms$i.json 2>/dev/null; done
echo done
