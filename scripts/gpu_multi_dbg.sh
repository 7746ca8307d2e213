mkdir -p gpurun_out/tr
N=$(nvidia-smi -L | wc -l)
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
    --log-dir gpurun_out/tr --redirects 3 --tee 3 bench.py --gpus $N --steps 5 --warmup 3 --workload cfg4 > gpurun_out/dbg_cfg4.json 2> gpurun_out/dbg_cfg4.err
echo "rc=$?" >> gpurun_out/dbg_cfg4.err
timeout 900 python -m pytest tests/test_gpu_multigpu.py -x -q > gpurun_out/pytest_multigpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_multigpu.log
echo done
