# batch / sweep GPU tests and a cfg5 bench line
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_price.py -x -q -m gpu > gpurun_out/pytest_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_sweep.log
timeout 600 python bench.py --workload cfg5 --steps 10 --warmup 3 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
echo done
