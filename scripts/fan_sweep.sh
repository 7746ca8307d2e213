mkdir -p gpurun_out
TP_PROFILE_HOST=1 python scripts/e2e_probe.py > gpurun_out/e2e.log 2>&1
python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
