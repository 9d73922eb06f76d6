mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_group.py -q -p no:cacheprovider -x > gpurun_out/pytest_group.log 2>&1; echo group_exit=$?
tail -n 2 gpurun_out/pytest_group.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 10 --warmup 3 --force-group --no-cpu-baseline > gpurun_out/bench_group.log 2>&1; echo groupbench_exit=$?
grep '^{' gpurun_out/bench_group.log | tail -n 1 | cut -c1-400
