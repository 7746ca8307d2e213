mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --workload cfg5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:fused \
  --csv --log-file gpurun_out/launches_cfg5.csv python bench.py --workload cfg5 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/ncu_l5.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:fused_batch --launch-skip 3 --launch-count 1 \
  -o gpurun_out/batch_full -f python bench.py --workload cfg5 --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/ncu_b5.log 2>&1
echo done
