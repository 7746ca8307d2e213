# N-GPU bench lines (torchrun, one process per GPU): the default line (cfg4 weak
# + the cfg5 block, strong) and the reference arm; the multi-GPU tests.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_multigpu.py -x -q > gpurun_out/pytest_multigpu_n$N.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_multigpu_n$N.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus $N > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --impl reference --gpus $N --steps 3 --warmup 3 > gpurun_out/bench_ref_n$N.json 2> gpurun_out/bench_ref_n$N.err
echo done
