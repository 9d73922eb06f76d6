for i in 1 2 3; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 2951$i bench.py --gpus 1 --steps 20 --warmup 5 --force-group --no-cpu-baseline > gpurun_out/bench_group.log 2>&1
python -c "import json; l=[x for x in open('gpurun_out/bench_group.log') if x.startswith('{')]; d=json.loads(l[-1]); print('group', d['ms_per_step'])"
done
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b.log 2>&1; python -c "import json; l=[x for x in open('gpurun_out/b.log') if x.startswith('{')]; d=json.loads(l[-1]); print('plain', d['ms_per_step'])"
