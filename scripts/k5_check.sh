timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_engine.py -q -m gpu -x 2>&1 | tail -2
timeout 900 python bench.py --steps 5 --warmup 3 --skip-cpu --skip-e2e > gpurun_out/k5_c2.log 2>&1; grep '^{' gpurun_out/k5_c2.log > gpurun_out/k5_c2.json; python scripts/line_summary.py gpurun_out/k5_c2.json 2>/dev/null | head -12
