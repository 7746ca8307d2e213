mkdir -p gpurun_out
TAG=${TAG:-r02j}
timeout 1200 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_multidevice.py -x -q > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}.log
TP_PROFILE_HOST=1 timeout 600 python bench.py --workload cfg5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cfg5_${TAG}.json 2> gpurun_out/cfg5_${TAG}.err
for C in 1 4 16; do TP_PROFILE_HOST=1 TP_SWEEP_CHUNKS=$C timeout 600 python bench.py --workload cfg5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/cfg5_c${C}_${TAG}.json 2> gpurun_out/cfg5_c${C}_${TAG}.err; done
echo done
