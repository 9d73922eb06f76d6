# GEMM tuner: candidate timings (ML_GEMM_TUNE_LOG=1) and step times over several fresh processes
ML_GEMM_TUNE_LOG=1 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-variants 2>&1 | grep "gemm tune" | sort | uniq | head -60
for i in 1 2 3 4; do timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-variants 2>/dev/null | python -c "
import sys,json; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
print('run $i', round(d['ms_per_step'],4), d['kernel_ms_per_step'].get('cublasLt_gemm'))"; done
