bash scripts/gpu_tc.sh
bash scripts/gpu_ncu_full2.sh
