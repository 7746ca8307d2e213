# run the fan-out probe against prebuilt engine variants in _variants/ (restores the in-tree build after)
mkdir -p gpurun_out; : > gpurun_out/variants.log
cp paper_2301_04285_b200/libtaps_b200.so /tmp/libtaps_b200.keep.so
for v in ${VARIANTS:-base memearly}; do
  cp _variants/$v.so paper_2301_04285_b200/libtaps_b200.so
  echo "== $v" >> gpurun_out/variants.log
  python scripts/fan_probe.py 2>&1 | grep "build\|pairs start" >> gpurun_out/variants.log
  python scripts/fan_probe.py 2>&1 | grep "build\|pairs start" >> gpurun_out/variants.log
  timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "cfg4_vs_oracle or configs_vs_oracle or random_graphs or edge_range" 2>&1 | tail -1 >> gpurun_out/variants.log
done
cp /tmp/libtaps_b200.keep.so paper_2301_04285_b200/libtaps_b200.so
