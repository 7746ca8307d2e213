mkdir -p gpurun_out
python scripts/fan_probe.py > gpurun_out/fan.log 2>&1
python scripts/fan_probe.py >> gpurun_out/fan.log 2>&1
python -m pytest tests/test_gpu_parity.py tests/test_gpu_adapter.py -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
