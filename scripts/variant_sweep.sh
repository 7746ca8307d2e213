# run the fan-out probe against prebuilt engine variants in _variants/ (restores the in-tree build after)
mkdir -p gpurun_out; : > gpurun_out/variants.log
cp paper_2301_04285_b200/libtaps_b200.so /tmp/libtaps_b200.keep.so
for v in ${VARIANTS:-base plain}; do
  cp _variants/$v.so paper_2301_04285_b200/libtaps_b200.so
  echo "== $v" >> gpurun_out/variants.log
  python scripts/fan_probe.py 2>&1 | grep "build\|pairs start" >> gpurun_out/variants.log
  python scripts/fan_probe.py 2>&1 | grep "build\|pairs start" >> gpurun_out/variants.log
done
cp /tmp/libtaps_b200.keep.so paper_2301_04285_b200/libtaps_b200.so
for w in 0 1; do
  echo "== TP_BATCH_WIDE=$w" >> gpurun_out/variants.log
  TP_BATCH_WIDE=$w python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(l['ms_per_step'], l['value'])" >> gpurun_out/variants.log
done
