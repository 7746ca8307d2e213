mkdir -p gpurun_out
TP_PROFILE_HOST=1 timeout 300 python scripts/sweep_probe.py 2>&1 | grep -v "tp host" > gpurun_out/sweep_probe.log
echo done
