mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
TP_PROFILE_HOST=1 timeout 300 python scripts/sweep_probe.py 2>&1 | grep -v "tp host" > gpurun_out/sweep_probe.log
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err
echo done
