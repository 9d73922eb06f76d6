mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv,noheader
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r2a_pytest_gpu.log 2>&1; echo pytest_exit=$?
tail -3 gpurun_out/r2a_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo smoke_exit=$?; tail -2 gpurun_out/r2a_smoke.log
timeout 600 python bench.py > gpurun_out/r2a_bench.log 2>gpurun_out/r2a_bench.err; echo bench_exit=$?; tail -c 3000 gpurun_out/r2a_bench.log
