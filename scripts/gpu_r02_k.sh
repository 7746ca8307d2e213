mkdir -p gpurun_out
TAG=${TAG:-r02k}
timeout 1200 python -m pytest tests/test_gpu_sweep.py -x -q > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}.log
TP_PROFILE_HOST=1 timeout 600 python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 4 > gpurun_out/cfg5_${TAG}.json 2> gpurun_out/cfg5_${TAG}.err
echo done
