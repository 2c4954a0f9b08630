mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multirank.py -q -rf --timeout 600 > gpurun_out/multirank.log 2>&1; echo "multirank rc=$?"
bash scripts/gpu_profile_cfg.sh c5 C5 "filter_kernel|enum_kernel|sub_kernel" 4
bash scripts/gpu_profile_cfg.sh c2 C2 "enum_kernel" 1
tail -3 gpurun_out/multirank.log
