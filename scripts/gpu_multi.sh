# N-GPU evidence (gpurun --gpus N): the multi-GPU tests (NCCL gather across processes; the
# single-process multi-device build), the default bench line under torchrun (cfg4 weak + the
# cfg5 block strong + ONE cfg4 build edge-sharded over the N GPUs), the cfg5 line, the reference arm.
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
TAG=${TAG:-r02}
timeout 900 python -m pytest tests/test_gpu_multigpu.py tests/test_gpu_multidevice.py -x -q > gpurun_out/pytest_multigpu_n${N}_${TAG}.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_multigpu_n${N}_${TAG}.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus $N > gpurun_out/bench_n${N}_${TAG}.json 2> gpurun_out/bench_n${N}_${TAG}.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513 \
  bench.py --gpus $N --workload cfg5 > gpurun_out/bench_cfg5_n${N}_${TAG}.json 2> gpurun_out/bench_cfg5_n${N}_${TAG}.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --impl reference --gpus $N --steps 3 --warmup 3 > gpurun_out/bench_ref_n${N}_${TAG}.json 2> gpurun_out/bench_ref_n${N}_${TAG}.err
echo done
