# sweep tests (incl. the pipelined one-shot), cfg5 bench, fan-per variants of the batch's second launch.
mkdir -p gpurun_out
TAG=${TAG:-r02h}
timeout 1200 python -m pytest tests/test_gpu_sweep.py tests/test_gpu_multidevice.py tests/test_export.py -x -q > gpurun_out/pytest_${TAG}.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_${TAG}.log
TP_PROFILE_HOST=1 timeout 600 python bench.py --workload cfg5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cfg5_${TAG}.json 2> gpurun_out/cfg5_${TAG}.err
cp paper_2301_04285_b200/libtaps_b200.so /tmp/keep.so
for v in 1 2 4; do
  cp _variants/bfp$v.so paper_2301_04285_b200/libtaps_b200.so
  timeout 600 python bench.py --workload cfg5 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/cfg5_fp${v}_${TAG}.json 2>/dev/null
done
cp /tmp/keep.so paper_2301_04285_b200/libtaps_b200.so
echo done
