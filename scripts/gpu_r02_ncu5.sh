# cfg5 batch kernel: one --set full capture with source lines, plus the multi-device tests on one GPU.
mkdir -p gpurun_out
TAG=${TAG:-r02c}
timeout 600 python -m pytest tests/test_gpu_multidevice.py -x -q > gpurun_out/pytest_multi_${TAG}.log 2>&1
CMD5="python bench.py --workload cfg5 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 3"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fused_batch --launch-skip 3 --launch-count 1 \
  -o gpurun_out/batch_${TAG} -f $CMD5 > gpurun_out/ncu_batch_${TAG}.log 2>&1
echo done
