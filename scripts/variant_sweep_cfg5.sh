# cfg5 batched build against prebuilt engine variants in _variants/ (restores the in-tree build after)
mkdir -p gpurun_out; : > gpurun_out/variants5.log
cp paper_2301_04285_b200/libtaps_b200.so /tmp/libtaps_b200.keep.so
for v in ${VARIANTS:-g8 g4 g16}; do
  cp _variants/$v.so paper_2301_04285_b200/libtaps_b200.so
  for i in 1 2; do
    echo "== $v" >> gpurun_out/variants5.log
    python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(l['ms_per_step'], l['value'], l['config']['build_ms_e2e'])" >> gpurun_out/variants5.log
  done
done
cp /tmp/libtaps_b200.keep.so paper_2301_04285_b200/libtaps_b200.so
