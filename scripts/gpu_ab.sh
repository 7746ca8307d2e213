# A/B of the fan-out (pairs of ids per thread vs one id): parity of the new build, then
# fan_probe + cfg5 + cfg4 bench on both prebuilt variants (_variants/base.so, _variants/lean.so).
mkdir -p gpurun_out
TAG=${TAG:-r02m}
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sweep.py tests/test_gpu_multidevice.py -x -q > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}.log
cp paper_2301_04285_b200/libtaps_b200.so /tmp/keep.so
: > gpurun_out/ab_${TAG}.log
for v in base rows base rows; do
  cp _variants/$v.so paper_2301_04285_b200/libtaps_b200.so
  echo "== $v" >> gpurun_out/ab_${TAG}.log
  python scripts/fan_probe.py 2>&1 | grep "build" >> gpurun_out/ab_${TAG}.log
  timeout 600 python bench.py --workload cfg5 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg5', d['ms_per_step'])" >> gpurun_out/ab_${TAG}.log
done
cp /tmp/keep.so paper_2301_04285_b200/libtaps_b200.so
echo done
