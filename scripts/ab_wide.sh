mkdir -p gpurun_out; : > gpurun_out/ab_wide.log
cp paper_2301_04285_b200/libtaps_b200.so /tmp/keep.so
run() { # name so wide
  cp _variants/$2.so paper_2301_04285_b200/libtaps_b200.so
  for i in 1 2; do
    echo "== $1" >> gpurun_out/ab_wide.log
    TP_BATCH_WIDE=$3 python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 3 2>/dev/null | python -c "import json,sys; l=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(l['ms_per_step'], l['value'])" >> gpurun_out/ab_wide.log
  done
}
run new new 0; run new_wide2 new 1; run w3_wide3 w3 1; run new new 0; run new_wide2 new 1; run w3_wide3 w3 1
cp /tmp/keep.so paper_2301_04285_b200/libtaps_b200.so
echo done
