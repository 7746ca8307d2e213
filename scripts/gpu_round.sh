# tests + bench + probe on one GPU (no ncu)
mkdir -p gpurun_out
python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench2.json 2> gpurun_out/bench2.err
python scripts/fan_probe.py > gpurun_out/fan.log 2>&1
echo done
