mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "strategies" > gpurun_out/pytest_strat.log 2>&1; echo strat_tests=$?
tail -5 gpurun_out/pytest_strat.log
timeout 1200 python scripts/bench_strategies.py > gpurun_out/strategies.jsonl 2>gpurun_out/strategies.err; echo bench_exit=$?
cat gpurun_out/strategies.jsonl | cut -c1-300; tail -3 gpurun_out/strategies.err
