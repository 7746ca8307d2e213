mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_adapter.py -x -q -s > gpurun_out/pytest_adapter.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_adapter.log
timeout 300 python scripts/fan_probe.py > gpurun_out/fan.log 2>&1
echo done
