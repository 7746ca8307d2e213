# run the probe against prebuilt engine variants in _variants/ (restores fan4)
mkdir -p gpurun_out; : > gpurun_out/variants.log
for v in ${VARIANTS:-fan2 fan4 fan6}; do
  cp _variants/$v.so paper_2301_04285_b200/libtaps_b200.so
  echo "== $v" >> gpurun_out/variants.log
  python scripts/fan_probe.py 2>&1 | grep build >> gpurun_out/variants.log
  python scripts/fan_probe.py 2>&1 | grep build >> gpurun_out/variants.log
done
