# A/B of prebuilt engine variants (_variants/*.so, git-ignored): parity tests of the in-tree
# build, then fan_probe.py (FAN=1) and the cfg5 bench (unless NO5=1) on each variant; VARIANTS picks them.
mkdir -p gpurun_out
TAG=${TAG:-ab}
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sweep.py tests/test_gpu_multidevice.py -x -q > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}.log
cp paper_2301_04285_b200/libtaps_b200.so /tmp/keep.so
: > gpurun_out/ab_${TAG}.log
for v in ${VARIANTS:-base new base new}; do
  cp _variants/$v.so paper_2301_04285_b200/libtaps_b200.so
  echo "== $v" >> gpurun_out/ab_${TAG}.log
  [ -n "$FAN" ] && python scripts/fan_probe.py 2>&1 | grep "^build " >> gpurun_out/ab_${TAG}.log
  [ -z "$NO5" ] && timeout 600 python bench.py --workload cfg5 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg5', d['ms_per_step'], d['config']['build_ms_e2e'])" >> gpurun_out/ab_${TAG}.log
done
cp /tmp/keep.so paper_2301_04285_b200/libtaps_b200.so
if [ -n "$NCU5" ]; then
  CMD5="python bench.py --workload cfg5 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 3"
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"batch|infer" -c 30 --csv \
    --log-file gpurun_out/launches_cfg5_${TAG}.csv $CMD5 > gpurun_out/ncu_launches5_${TAG}.log 2>&1
fi
echo done
