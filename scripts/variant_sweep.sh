# run the fan-out probe against prebuilt engine variants in _variants/ (restores the in-tree build after)
mkdir -p gpurun_out; : > gpurun_out/variants.log
cp paper_2301_04285_b200/libtaps_b200.so /tmp/libtaps_b200.keep.so
for v in ${VARIANTS:-base static}; do
  cp _variants/$v.so paper_2301_04285_b200/libtaps_b200.so
  echo "== $v" >> gpurun_out/variants.log
  python scripts/fan_probe.py 2>&1 | grep "build\|pairs start" >> gpurun_out/variants.log
  python scripts/fan_probe.py 2>&1 | grep "build\|pairs start" >> gpurun_out/variants.log
done
cp /tmp/libtaps_b200.keep.so paper_2301_04285_b200/libtaps_b200.so

