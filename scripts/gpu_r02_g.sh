mkdir -p gpurun_out
TAG=${TAG:-r02g}
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}.log
python scripts/class_probe.py > gpurun_out/class_${TAG}.log 2>&1
python scripts/fan_probe.py > gpurun_out/fan_${TAG}.log 2>&1
timeout 600 python bench.py --workload cfg5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cfg5_${TAG}.json 2> gpurun_out/cfg5_${TAG}.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-sweep --no-configs --no-cpu-baseline > gpurun_out/cfg4_${TAG}.json 2> gpurun_out/cfg4_${TAG}.err
echo done
